/*
 * hive_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, sequential, slow CPU implementation of the Hive hash table
 * (arXiv 2510.15095, reference/PAPER.md) used to check the CUDA path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  It shares no code, header, table or
 * constant with paper_2510_15095_b200/ (the product), and the product never
 * loads it.
 *
 * Every function cites the PAPER.md line (section / algorithm / listing) it
 * follows; readings of silent or garbled passages are the A-n items of
 * SURVEY.md Appendix A, restated in DESIGN.md "Readings".
 */
#ifndef HIVE_ORACLE_H
#define HIVE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_table* oracle_t;

typedef struct {
    uint64_t n_buckets;      /* 2^m + split                                  */
    uint32_t m;              /* round level, index_mask = 2^m - 1 */
    uint32_t split;          /* split pointer                    */
    uint64_t count;          /* live keys, buckets + stash (reading A-19)    */
    uint64_t stash_live;     /* live stash entries                           */
    uint64_t stash_cap;      /* ring capacity (reading A-8)                  */
    uint64_t step1;          /* inserts completed by Step 1 (replace)        */
    uint64_t step2;          /* inserts completed by Step 2 (claim)          */
    uint64_t step3_entries;  /* inserts that entered Step 3                  */
    uint64_t step3_ok;       /* ... and were placed by Step 3                */
    uint64_t step3_rounds;   /* total Step-3 rounds (kicks)                  */
    uint64_t step4;          /* stash pushes (Step 4)                        */
    uint64_t lock_acq;       /* Alg. 3 bucket-lock acquisitions              */
    uint64_t max_depth;      /* deepest Step-3 round count of one insert     */
    uint64_t grows;          /* expand_batch calls                           */
    uint64_t shrinks;        /* contract_batch calls                         */
    uint64_t merge_aborts;   /* aborted merges                               */
    uint64_t pending;        /* stash-full entries (must stay 0)             */
    uint64_t in_b1;          /* live bucket keys resident in addr(h1)        */
} oracle_stats_t;

/* Table lifecycle (§III-B; sizing per SURVEY §8(b)). */
oracle_t oracle_create(uint64_t capacity_slots, uint64_t max_capacity_slots,
                       float lf_grow, float lf_shrink, uint32_t max_evictions,
                       uint32_t resize_k, float stash_fraction);
void     oracle_destroy(oracle_t t);

/* Batch operations under the PHASED contract. Return 0 on
 * success, nonzero if an invariant-breaking event (stash full) happened. */
int oracle_insert(oracle_t t, const uint32_t* keys, const uint32_t* vals,
                  uint64_t n, uint8_t* status);
int oracle_find(oracle_t t, const uint32_t* keys, uint64_t n,
                uint32_t* vals_out, uint8_t* found);
int oracle_erase(oracle_t t, const uint32_t* keys, uint64_t n, uint8_t* erased);
int oracle_mixed(oracle_t t, const uint8_t* op, const uint32_t* keys,
                 const uint32_t* vals, uint64_t n, uint32_t* vals_out,
                 uint8_t* result);

void     oracle_get_stats(oracle_t t, oracle_stats_t* out);
uint64_t oracle_dump(oracle_t t, uint32_t* keys, uint32_t* vals, uint64_t cap);
/* Self-checks of SURVEY §8(c) "Oracle self-checks"; 0 = all hold. */
int      oracle_check(oracle_t t, char* msg, int msglen);

/* Direct resize hooks for fixtures. Return 1 if a merge
 * aborted. */
void oracle_expand(oracle_t t, uint32_t k);
int  oracle_contract(oracle_t t, uint32_t k);
/* Raw bucket view for fixtures: 32 slot words + freeMask. */
uint32_t oracle_bucket(oracle_t t, uint64_t b, uint64_t* slots32);
/* Bucket array (n_buckets * 32 words, may be NULL) and up to stash_cap live
 * stash words (may be NULL); returns the number of live stash entries. */
uint64_t oracle_image(oracle_t t, uint64_t* slots, uint64_t* stash, uint64_t stash_cap);

/* Primitives exposed so the pins can test them individually. */
uint64_t oracle_pack(uint32_t key, uint32_t value);
uint32_t oracle_unpack_key(uint64_t pair);
uint32_t oracle_unpack_value(uint64_t pair);
uint32_t oracle_bithash1(uint32_t key);
uint32_t oracle_bithash2(uint32_t key);
/* Lookup-based hashes of §V-B (reading A-26). */
uint32_t oracle_crc32_bytes(const uint8_t* p, uint64_t n);   /* CRC-32/IEEE */
uint64_t oracle_crc64_bytes(const uint8_t* p, uint64_t n);   /* CRC-64/XZ   */
uint32_t oracle_crc32(uint32_t key);      /* over the 4 LE key bytes        */
uint32_t oracle_crc64_lo(uint32_t key);   /* low 32 bits, 4 LE key bytes    */
/* Select the table's hash pair (0 BitHash1/2, 1 CRC-32/CRC-64) on an empty
 * table; nonzero return = refused. */
int oracle_set_hash(oracle_t t, uint32_t kind);
/* Theorem 1 and CSR. */
double   oracle_uniform_expected_collisions(uint64_t n, uint64_t m);
uint64_t oracle_observed_collisions(uint32_t fn, const uint32_t* keys, uint64_t n, uint64_t m);
uint32_t oracle_addr(uint32_t h, uint32_t index_mask, uint32_t split);
uint32_t oracle_alt(uint32_t key, uint32_t cur, uint32_t index_mask, uint32_t split);
uint32_t oracle_ballot(const uint8_t* preds32);
int      oracle_first_set(uint32_t mask);
uint32_t oracle_prefix_rank(uint32_t mask, uint32_t lane);
int      oracle_select_nth_one(uint32_t mask, uint32_t r);
/* Shard of a key for the hash-partitioned table. */
uint32_t oracle_shard(uint32_t key, uint32_t seed, uint32_t n_shards);

#ifdef __cplusplus
}
#endif
#endif
