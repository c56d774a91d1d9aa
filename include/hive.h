/*
 * hive.h — C ABI of the B200-native Hive hash table (arXiv 2510.15095).
 *
 * The data-parallel hot path of the paper — batched, warp-cooperative insert /
 * lookup / delete over a packed bucket array of 64-bit key-value words, WABC
 * slot claiming, WCME matching, the four-step insert, and load-factor-triggered
 * linear-hashing split/merge — implemented as hand-written sm_100a CUDA in
 * libhive.so.  No torch types appear here: all arguments are plain integers and
 * pointers.  Citations: PAPER:L = reference PAPER.md line; SURVEY §x = the
 * blueprint section; A-n = reading n of DESIGN.md "Readings of the paper".
 *
 * Conventions for every call
 *  - d_* arguments are DEVICE pointers owned by the caller; they must stay
 *    alive until the work on `stream` completes.  h_* are HOST pointers.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Calls are stream-ordered and asynchronous unless noted "sync".
 *  - Keys and values are uint32.  Key 0xFFFFFFFF is reserved (it encodes the
 *    EMPTY slot word, A-9): insert reports status 2, find reports not-found,
 *    erase reports 0 for it.
 *  - n == 0 is a no-op returning HIVE_OK.
 *  - A handle is used by one stream at a time (phases never overlap); a call
 *    made while another call on the same handle is still being issued returns
 *    HIVE_EBUSY.  Different handles are independent.
 *  - Errors: argument errors return immediately without launching work
 *    (HIVE_EINVAL); CUDA errors map to HIVE_ECUDA with the text available from
 *    hive_last_error(); a stash overflow (never expected at LF <= 0.95) sets
 *    per-op status 3 and a sticky flag reported by hive_stats / hive_size as
 *    HIVE_ESTASHFULL.
 *
 * Batch semantics (PHASED contract): a batch applies all INSERT
 * ops, then all ERASE ops, then all FIND ops.  Insert status and erase output
 * are present(k) at the start of their phase and identical for in-batch
 * duplicates; after an insert phase k holds the value of the LAST op (highest
 * index) inserting k in the batch — one member of the accepted set.  Find
 * returns (present, value) at the FIND-phase start.  Resize happens only at
 * phase boundaries: grow before INSERT while count + n_ins > lf_grow * slots
 * (PAPER:482), shrink after ERASE while count < lf_shrink * slots.
 */
#ifndef HIVE_H
#define HIVE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hive_table_s* hive_t;

typedef enum {
    HIVE_OK = 0,
    HIVE_EINVAL = 1,      /* bad argument / config                          */
    HIVE_ENOMEM = 2,      /* device or VA allocation failed                 */
    HIVE_ECUDA = 3,       /* CUDA runtime / driver error                    */
    HIVE_ENCCL = 4,       /* NCCL error (sharded tables)                    */
    HIVE_ESTASHFULL = 5,  /* sticky: an entry could not be stored           */
    HIVE_EBUSY = 6,       /* handle already in use by a concurrent call     */
    HIVE_EXCHANGE = 7     /* sticky (sharded): an op did not fit its padded
                             exchange region and was not processed          */
} hive_status;

/* Flags for hive_config.flags */
#define HIVE_KEYS_UNIQUE 1u   /* caller asserts: no duplicate keys inside any one
                                 insert or erase batch -> the owner-election
                                 pass is skipped.  Results
                                 are undefined if the assertion is false. */
#define HIVE_HASH_CRC    2u   /* use the lookup-based hash pair of §V-B
                                 (PAPER:569-574): h1 = CRC-32/IEEE, h2 = low 32
                                 bits of CRC-64/XZ, over the 4 little-endian key
                                 bytes, byte-wise tables read through the L1 read-only path
                                 (reading A-26).  Default (flag clear):
                                 BitHash1 / BitHash2 (Listing 1).  Any other
                                 flag bit -> HIVE_EINVAL. */
#define HIVE_SHARD_DEDUP 4u   /* sharded handles only: elect one owner per (key,
                                 opcode) among each rank's local batch before
                                 routing (SURVEY §8(e) Zipf item); only owners
                                 are exchanged and the other ops copy their
                                 owner's result.  Results are unchanged; under
                                 skewed keys the hot key's region holds one
                                 record per rank instead of all its copies.
                                 Costs one election pass over the local batch.
                                 Requires nccl_comm and shard_batch_max < 2^30. */

typedef struct {
    uint64_t capacity;       /* initial slots; rounded up to 32-slot buckets
                                (>= 2 buckets); any count (A-20)              */
    uint64_t max_capacity;   /* slots reserved (virtual) for growth; 0 = half
                                of device memory                             */
    float    lf_grow;        /* 0.90; >= 1.0 disables growth      */
    float    lf_shrink;      /* 0.25; <= 0 disables contraction   */
    uint32_t max_evictions;  /* Step-3 bound, 16 (value A-8)       */
    uint32_t resize_k;       /* K buckets per split/merge batch, 1024
                                (value A-8)                        */
    float    stash_fraction; /* stash capacity / slots, 0.02,
                                floor 1024 entries                           */
    uint32_t flags;          /* HIVE_KEYS_UNIQUE | HIVE_HASH_CRC              */
    /* ---- sharded tables ---- */
    void*    nccl_comm;      /* NULL: single-GPU table.  Else an ncclComm_t
                                (e.g. from hive_nccl_comm_init): this handle is
                                rank `rank` of a hash-partitioned table of
                                `nranks` shards (rank and size from the comm);
                                capacity etc. are PER SHARD.  Owned by the
                                caller; must outlive the handle.              */
    uint64_t shard_batch_max;/* sharded: the largest local batch any rank
                                passes to one call (required, > 0)            */
    float    shard_slack;    /* sharded: padded exchange capacity per peer =
                                ceil(shard_batch_max / nranks * (1 + slack))
                                + 1024 records; default 0.0625              */
} hive_config;

/* Stats snapshot (sync). */
typedef struct {
    uint64_t n_buckets;      /* 2^m + split_ptr                               */
    uint32_t m;              /* round level; index_mask = 2^m - 1 */
    uint32_t split;          /* split pointer                     */
    uint64_t count;          /* live keys (buckets + stash)                   */
    uint64_t stash_used;     /* stash ring slots used since the last drain    */
    uint64_t stash_cap;      /* stash ring capacity                           */
    uint64_t evictions;      /* Step-3 victim swaps, cumulative               */
    uint64_t max_depth;      /* deepest Step-3 round count of one insert      */
    uint64_t stash_pushes;   /* Step-4 pushes, cumulative                     */
    uint64_t leftovers;      /* inserts that reached Step 3, cumulative       */
    uint64_t grows;          /* split batches run                             */
    uint64_t shrinks;        /* merge batches run                             */
    uint64_t merge_aborts;   /* merges aborted for lack of space  */
    uint64_t failed;         /* entries lost to a full stash (must be 0)      */
    uint64_t in_b1;          /* live bucket keys resident in addr(h1)         */
    uint64_t mapped_bytes;   /* physical bytes mapped for buckets             */
    uint64_t alg_bytes[8];   /* algorithmic bytes touched since create/clear,
                                per kernel family: [0] find, [1] insert fast
                                path, [2] eviction + stash, [3] erase,
                                [4] owner election (256 B per bucket probe,
                                32 B per CAS sector, 8 B per spill / stash
                                word, exact key / value / result stream
                                bytes)                          */
    uint64_t step3;          /* entries placed by the Step-3 loop (new keys,
                                reinserted stash entries, lost fast claims);
                                Step-2 placements = new keys - leftovers      */
    uint64_t xfail;          /* sharded: ops of this rank not processed
                                because their exchange region was full        */
    uint64_t elect_overflow; /* owner-election table overflows (must be 0: the
                                tables hold 2.5x the mean part size)          */
    uint64_t step_cycles[4]; /* insertion step breakdown,
                                collected while hive_profile level 2 is on:
                                warp clock64() cycles in Step 1 (replace),
                                Step 2 (claim-and-commit), Step 3 (bounded
                                eviction), Step 4 (stash fallback); per warp
                                region max-over-lanes end minus min-over-lanes
                                start, summed over warps and regions          */
} hive_stats_t;

/* ---- Sharded tables (BASELINE configs[4]) ---------------
 * A handle created with cfg.nccl_comm != NULL is one shard of a table
 * hash-partitioned over the comm's ranks: key k is owned by rank
 * shard(k) = (fmix32(k ^ HIVE_SHARD_SEED) * nranks) >> 32 (MurmurHash3's
 * finaliser, independent of BitHash1/2 so every shard uses all its buckets).
 * Every op call (hive_insert / find / erase / mixed and their _host forms) is
 * COLLECTIVE: all ranks call it in the same order, each with its own local
 * batch (n may differ per rank, 0 allowed, n <= shard_batch_max), and each
 * gets the results for its own ops in its own order.  Semantics are those of
 * ONE single-GPU call on the union batch in (rank, index) order: e.g. among
 * in-batch duplicates the op of the highest (rank, index) wins.
 * Exchange: a stable route kernel packs each op record into a padded send
 * buffer of nranks regions of C = shard_slack-padded capacity, then one
 * ncclAlltoAll moves the per-region counts and one the records (plus one
 * for opcodes in mixed calls); each owner compacts the received records by
 * device-side counts and runs the PHASED batch; results return by the inverse
 * ncclAlltoAll and an unpermute kernel.  No host synchronisation happens when
 * growth and contraction are off (lf_grow >= 1, lf_shrink <= 0), so the whole
 * call can be captured in a CUDA graph.  An op that does not fit its region
 * (more than C ops of one rank's batch owned by one shard -- a ~30-sigma
 * event for hashed keys at the default slack) is not processed: insert /
 * erase / mixed result 4, find found = 2, and the handle's sticky
 * HIVE_EXCHANGE flag is reported by hive_stats / hive_size.
 * hive_clear / size / stats / dump / profile act on the local shard only. */
#define HIVE_SHARD_SEED 0x5BD1E995u

/* NCCL bootstrap without NCCL headers in the caller (libnccl.so.2 is loaded
 * at run time; ncclAlltoAll needs NCCL >= 2.28, older versions use grouped
 * send / recv).  hive_nccl_unique_id (rank 0) fills 128 bytes that the caller
 * broadcasts to every rank (e.g. through torch.distributed); every rank then
 * calls hive_nccl_comm_init with the current CUDA device set (collective).
 * hive_nccl_comm_destroy frees a comm made here.  HIVE_ENCCL on failure. */
hive_status hive_nccl_unique_id(uint8_t* id_out);
hive_status hive_nccl_comm_init(int nranks, int rank, const uint8_t* id, void** comm_out);
hive_status hive_nccl_comm_destroy(void* comm);
/* Shard geometry of a handle: *nranks = 1, *rank = 0 for a single-GPU table. */
hive_status hive_shard_info(hive_t h, int* nranks, int* rank, uint64_t* cap_per_peer);

/* Fill *cfg with the defaults above. */
void hive_config_default(hive_config* cfg);

/* Create a table (sync).  Reserves virtual address space for max_capacity
 * and maps physical 2 MiB chunks for the initial buckets (EMPTY-filled).
 * Returns HIVE_EINVAL for cfg == NULL, out == NULL, capacity == 0,
 * lf_shrink >= lf_grow (when both are enabled), stash_fraction < 0, or a
 * sharded config with shard_batch_max == 0, more than 32 ranks or a padded
 * exchange of 2^32 records or more; HIVE_ENCCL if the comm cannot be queried.
 * Sharded: collective (no communication, but every rank must create its
 * shard before the first op call). */
hive_status hive_create(const hive_config* cfg, void* stream, hive_t* out);

/* Destroy (sync on the table's last stream); frees everything it owns. */
hive_status hive_destroy(hive_t h);

/* Four-step insert / replace.  d_keys, d_vals: uint32[n].
 * d_status (nullable): uint8[n]; 0 = absent at phase start (inserted),
 * 1 = present (value replaced), 2 = reserved key, 3 = this op's eviction
 * chain found the stash full and dropped its in-hand entry (this key or a key
 * it displaced; hive_stats.failed counts dropped entries, reading A-28),
 * 4 = not processed (sharded handles only: exchange region full).
 * May grow the table first (one small D2H of the counters when growth is
 * enabled). */
hive_status hive_insert(hive_t h, const uint32_t* d_keys, const uint32_t* d_vals,
                        uint64_t n, uint8_t* d_status, void* stream);

/* Lookup by WCME over the two candidate buckets, then the stash index
 * (PAPER:444-445).  d_vals_out: uint32[n] (value or 0 when absent);
 * d_found (nullable): uint8[n] 1/0. */
hive_status hive_find(hive_t h, const uint32_t* d_keys, uint64_t n,
                      uint32_t* d_vals_out, uint8_t* d_found, void* stream);

/* Delete (Alg. 4).  d_erased (nullable): uint8[n], 1 if the
 * key was present at phase start.  May shrink the table afterwards. */
hive_status hive_erase(hive_t h, const uint32_t* d_keys, uint64_t n,
                       uint8_t* d_erased, void* stream);

/* Mixed batch: d_op uint8[n] with 0 = find, 1 = insert, 2 = erase (other
 * codes: result 0).  Runs INSERT, ERASE, FIND phases.
 * d_vals_out uint32[n]: find value (0 for misses and non-find ops);
 * d_result uint8[n]: the op's own status code as above. */
hive_status hive_mixed(hive_t h, const uint8_t* d_op, const uint32_t* d_keys,
                       const uint32_t* d_vals, uint64_t n, uint32_t* d_vals_out,
                       uint8_t* d_result, void* stream);

/* Monolithic concurrent mixed batch (the paper's
 * single-kernel model): the whole batch runs in ONE
 * cooperative kernel launch, finds, erases and inserts interleaved in the same
 * pass (no opcode classification, no phases).  Arguments and result codes are
 * those of hive_mixed.  Contract (differs from hive_mixed's PHASED order):
 * per key, all insert ops of the batch form one insert group and all erase
 * ops one erase group; each group takes effect as one atomic step (its owner,
 * the highest op index, applies it; an insert group stores its owner's
 * value) and every member reports the key's presence before that step; each
 * find is its own atomic read.  The results are LINEARIZABLE per key: some
 * order of {insert group, erase group, finds} explains every result and the
 * final table.  Single-type batches therefore give exactly hive_insert /
 * hive_erase / hive_find's results.  Evictions (Step 3) run at the tail of
 * the same launch, after every find and erase, so no lookup observes an
 * entry held by an eviction chain (reading A-16).  Growth before the batch
 * and contraction after it follow hive_mixed's rule (one wait when growth or
 * contraction is enabled).  n < 2^31.  HIVE_EINVAL on sharded handles. */
hive_status hive_mixed_concurrent(hive_t h, const uint8_t* d_op, const uint32_t* d_keys,
                                  const uint32_t* d_vals, uint64_t n, uint32_t* d_vals_out,
                                  uint8_t* d_result, void* stream);

/* Host-buffer variants (the end-to-end public path).  h_* are HOST pointers
 * (page-locked memory recommended; pageable works but serialises copies).
 * Stream-ordered like the device calls: the results are in the host buffers
 * once `stream` has completed the call, and the host buffers must stay alive
 * until then.  Semantics are those of hive_insert / hive_find.  Internally the
 * transfers run on the handle's own upload / download streams in 4 Mi-op
 * chunks so that copies overlap compute: the owner election starts once all
 * keys are on the device and overlaps the value upload, insert chunks start as
 * their values land, find chunks overlap the download of earlier results, and
 * a find's upload may overlap a preceding insert's compute.  Device staging
 * buffers are owned by the handle (allocated on first use, reused). */
hive_status hive_insert_host(hive_t h, const uint32_t* h_keys, const uint32_t* h_vals,
                             uint64_t n, uint8_t* h_status, void* stream);
hive_status hive_find_host(hive_t h, const uint32_t* h_keys, uint64_t n,
                           uint32_t* h_vals_out, uint8_t* h_found, void* stream);

/* Reset to the freshly created state (all slots EMPTY, initial size, stash
 * empty, counters zero); keeps allocations.  Async. */
hive_status hive_clear(hive_t h, void* stream);

/* Live key count (sync). */
hive_status hive_size(hive_t h, uint64_t* out);

/* Stats snapshot (sync); returns HIVE_ESTASHFULL if the sticky flag is set. */
hive_status hive_stats(hive_t h, hive_stats_t* out);

/* Export all live pairs (sync) into caller DEVICE buffers of capacity cap
 * (order unspecified).  *n_out = number of live pairs (may exceed cap, in
 * which case only cap are written). */
hive_status hive_dump(hive_t h, uint32_t* d_keys, uint32_t* d_vals, uint64_t cap,
                      uint64_t* n_out, void* stream);

/* Test hook (sync): replace the table's contents with an
 * externally built image -- e.g. the CPU oracle's layout -- so that the probe
 * kernels can be checked against a layout the GPU insert path did not make.
 * d_slots: DEVICE uint64[n_buckets * 32] packed words (EMPTY = all ones) in
 * bucket order; the geometry becomes (m = floor(log2 n_buckets), split =
 * n_buckets - 2^m) with the Litwin addressing of PAPER:485-503 (A-2).
 * d_stash: DEVICE uint64[n_stash] live stash words (nullable when 0); the
 * stash capacity follows n_buckets.  Spill words and the stash index are
 * rebuilt, count = live slots + n_stash, statistics reset.  Every key must sit
 * in one of its candidate buckets or the stash, once (not checked).
 * HIVE_EINVAL for n_buckets < 2 or above max_capacity, n_stash above the
 * stash capacity, or a sharded handle. */
hive_status hive_load_image(hive_t h, const uint64_t* d_slots, uint64_t n_buckets, const uint64_t* d_stash,
                            uint64_t n_stash, void* stream);

/* Per-kernel device timing (CUDA events around every launch on the call's
 * stream).  Enabled by hive_profile(h, 1); hive_profile(h, 2) additionally
 * runs the insert kernels' clock64-instrumented variants (default lane
 * geometry) that fill hive_stats.step_cycles.  hive_profile_read fills up to
 * max entries of names (pointers to static strings), total milliseconds and
 * launch counts, returns the number of kernels seen, and resets when
 * reset != 0.  Sync. */
hive_status hive_profile(hive_t h, int enable);
int hive_profile_read(hive_t h, const char** names, double* ms, uint64_t* launches,
                      int max, int reset);

/* ---- stable partition (routing a batch across hash-partitioned shards,
 * SURVEY §8(e)); hive_mixed classifies its ops with a separate one-pass,
 * order-free kernel -------------------------------------------------------- */

/* Route a batch to n_shards shards: shard(k) = (fmix32(k ^ seed) * n_shards)
 * >> 32.  Stable (rank order preserved inside each shard).
 *   d_keys, d_vals (nullable), d_ops (nullable): the batch, length n.
 *   d_send_kv: uint64[n] packed (value << 32 | key) in shard order;
 *   d_send_ops (nullable): uint8[n] in shard order;
 *   d_pos: uint32[n], d_pos[i] = position of op i in the send buffer;
 *   d_counts: uint64[n_shards] ops per shard.
 * n_shards in [1, 64].  n must be < 2^32. */
hive_status hive_route(uint32_t n_shards, uint32_t seed, const uint32_t* d_keys,
                       const uint32_t* d_vals, const uint8_t* d_ops, uint64_t n,
                       uint64_t* d_send_kv, uint8_t* d_send_ops, uint32_t* d_pos,
                       uint64_t* d_counts, void* stream);

/* Keys-only variant for find / erase batches: d_send_keys uint32[n] in shard
 * order (half the bytes of the packed records, no unpack pass). */
hive_status hive_route_keys(uint32_t n_shards, uint32_t seed, const uint32_t* d_keys, uint64_t n,
                            uint32_t* d_send_keys, uint32_t* d_pos, uint64_t* d_counts, void* stream);

/* Inverse permutation gather after the results come back:
 * d_out8[i] = d_in8[d_pos[i]] and d_out32[i] = d_in32[d_pos[i]]
 * (either pair may be NULL). */
hive_status hive_unroute(const uint32_t* d_pos, uint64_t n, const uint8_t* d_in8,
                         uint8_t* d_out8, const uint32_t* d_in32, uint32_t* d_out32,
                         void* stream);

/* ---- peer-memory exchange -------------------------
 * The sharded table's exchange without NCCL: source ranks store op records
 * straight into the owners' inboxes and owners store results straight back,
 * over NVLink peer mappings (CUDA IPC).  1 <= n_shards <= 8.  Every exchange
 * buffer is laid out in `region`-sized regions, one per rank:
 *   inbox_kv  uint64[n_shards * region]  owner side; source r writes
 *             (value << 32 | key) records at [r * region, r * region + cnt[r])
 *   inbox_ops uint8 [n_shards * region]  same layout, opcodes (mixed batches)
 *   cnt       uint64[n_shards]           owner side; cnt[r] written by source r
 *   res32/res8 [n_shards * region]       source side; owner o writes results at
 *             [o * region, ...) in the order it received them
 * Peer pointer arguments are HOST arrays of n_shards DEVICE pointers (entry
 * p = shard p's buffer as mapped in this process; this rank's own entry is its
 * local buffer).  The caller orders the phases: route on every rank, a
 * cross-rank barrier (stream sync + process-group barrier), compact + the
 * owner's batch op + return, a barrier, then hive_unroute(d_pos, ...) over
 * res8 / res32 gives results in the caller's op order.  n_shards * region
 * must be <= 2^32 (positions are 32-bit). */

/* Stable route of this rank's batch into the owners' inboxes (shard(k) as in
 * hive_route), then cnt[rank] on every owner (records stored, <= region).
 * d_pos uint32[n]: p * region + (position in this rank's region of owner p),
 * the hive_unroute index into res8 / res32; an op past its region's capacity
 * is not sent and gets d_pos = 0xFFFFFFFF (use hive_unroute_pad).  d_counts
 * uint64[n_shards]: ops per owner before clipping (device).  d_ops / peer_ops
 * nullable together. */
hive_status hive_route_p2p(uint32_t n_shards, uint32_t rank, uint32_t seed, const uint32_t* d_keys,
                           const uint32_t* d_vals, const uint8_t* d_ops, uint64_t n, uint64_t region,
                           uint64_t* const* peer_kv, uint8_t* const* peer_ops, uint64_t* const* peer_cnt,
                           uint32_t* d_pos, uint64_t* d_counts, void* stream);
/* Owner, device-count form (no host synchronisation): compact the n_src inbox
 * regions by the device counts d_cnt, run this handle's op of `kind`
 * (0 find, 1 insert, 2 erase, 3 mixed: opcodes from d_inbox_ops) on the union
 * batch in source-rank order, and store every result straight into its
 * source's result region (peer_res32 for find / mixed, peer_res8 always).
 * Scratch (18 B per inbox record) is owned by the handle, grown on first use.
 * The host waits only if the op itself needs a count (growth / contraction
 * enabled).  HIVE_EINVAL on sharded (NCCL) handles. */
hive_status hive_serve_inbox(hive_t h, uint32_t kind, uint32_t n_src, uint32_t rank, uint64_t region,
                             const uint64_t* d_inbox_kv, const uint8_t* d_inbox_ops, const uint64_t* d_cnt,
                             uint32_t* const* peer_res32, uint8_t* const* peer_res8, void* stream);
/* hive_unroute for a route that can leave ops unsent (region capacity):
 * pos == 0xFFFFFFFF gives out8 = miss8 and out32 = 0.  d_poison (nullable):
 * a device word -- the peer exchange's timeout marker -- that, when non-zero
 * at execution time, turns every out8 into 6 (peer lost) and out32 into 0,
 * so results of an exchange that timed out are never returned as valid
 * without a host synchronisation. */
hive_status hive_unroute_pad(const uint32_t* d_pos, uint64_t n, const uint8_t* d_in8, uint8_t* d_out8,
                             const uint32_t* d_in32, uint32_t* d_out32, uint8_t miss8, const uint64_t* d_poison,
                             void* stream);
/* Owner: concatenate the n_src inbox regions (cnt[r] records each, rank order)
 * into d_keys / d_vals / d_ops [n_total = sum cnt] (d_ops with d_inbox_ops). */
hive_status hive_inbox_compact(uint32_t n_src, uint64_t region, const uint64_t* d_inbox_kv,
                               const uint8_t* d_inbox_ops, const uint64_t* d_cnt, uint64_t n_total,
                               uint32_t* d_keys, uint32_t* d_vals, uint8_t* d_ops, void* stream);
/* Owner: result j of the compacted batch (source r = the region j came from)
 * is stored at peer_res32[r][rank * region + (j - start_r)] (and res8). */
hive_status hive_return_p2p(uint32_t n_src, uint32_t rank, uint64_t region, const uint64_t* d_cnt,
                            uint64_t n_total, const uint32_t* d_res32, const uint8_t* d_res8,
                            uint32_t* const* peer_res32, uint8_t* const* peer_res8, void* stream);
/* Device-side phase barrier (replaces a host barrier between the phases).
 * Signal words: uint64[17] per rank, zeroed at allocation: [phase * 8 + r] =
 * the last epoch source r signalled for that phase, [16] = timeout marker.
 * hive_p2p_signal: after this rank's earlier stream work, store `epoch` into
 * every peer's word [phase * 8 + rank] (release, system scope).
 * hive_p2p_wait: stream-ordered wait until d_sig[phase * 8 + r] >= epoch for
 * all r < n (acquire); after timeout_ns it stops waiting and sets d_sig[16]
 * = 1, which the caller checks at its next synchronisation.  phase in {0, 1}. */
hive_status hive_p2p_signal(uint32_t n, uint32_t rank, uint32_t phase, uint64_t epoch,
                            uint64_t* const* peer_sig, void* stream);
hive_status hive_p2p_wait(uint32_t n, uint32_t phase, uint64_t epoch, uint64_t* d_sig, uint64_t timeout_ns,
                          void* stream);
/* Exchange buffers: plain cudaMalloc allocations (IPC-exportable base
 * pointers); the handle is the 64-byte cudaIpcMemHandle_t.  hive_ipc_open
 * maps a peer's buffer (peer access enabled lazily); hive_ipc_close unmaps. */
hive_status hive_dev_alloc(uint64_t bytes, void** d_out);
hive_status hive_dev_free(void* d_ptr);
hive_status hive_ipc_handle(const void* d_ptr, uint8_t* handle_out);
hive_status hive_ipc_open(const uint8_t* handle, void** d_out);
hive_status hive_ipc_close(void* d_ptr);

/* ---- hash study (§III-C Listing 1 / Theorem 1 / CSR, §V-B pairs) -------------
 * Hash functions by id: BitHash1 / BitHash2 (Listing 1), CRC-32
 * (IEEE) and the low 32 bits of CRC-64 (XZ), both over the 4 little-endian key
 * bytes from 256-entry tables (reading A-26; read-only L1 path, not constant memory). */
#define HIVE_FN_BITHASH1 0u
#define HIVE_FN_BITHASH2 1u
#define HIVE_FN_CRC32    2u
#define HIVE_FN_CRC64    3u
/* d_out[i] = fn(d_keys[i]) for i < n (device arrays, caller-owned; async on
 * `stream`).  HIVE_EINVAL for an unknown fn or null pointers with n > 0. */
hive_status hive_hash(uint32_t fn, const uint32_t* d_keys, uint64_t n, uint32_t* d_out,
                      void* stream);
/* Observed collisions Y = sum_b (L_b - 1)_+ of the n device keys over m
 * single-slot bins, bin = fn(k) mod m (Theorem 1; CSR =
 * E[Y] / Y).  Synchronous; *y_out is a host word.  Uses a
 * temporary m-bit device bitmap.  1 <= m <= 2^32, else HIVE_EINVAL. */
hive_status hive_collisions(uint32_t fn, const uint32_t* d_keys, uint64_t n, uint64_t m,
                            uint64_t* y_out, void* stream);

/* ---- calibration ceiling ------------------------------------
 * The pure gather a probe reduces to, timed beside the probe kernels: for
 * i < n, d_out[i] = xor of the 64 32-bit words of 256 B block
 * b = (fmix32(d_keys[i]) * n_blocks) >> 32 of d_blocks, read with the same
 * lane groups and 256-bit loads as the lookup kernel.  d_blocks: device,
 * 256 B aligned, n_blocks * 256 B; d_keys uint32[n], d_out uint32[n] device,
 * caller-owned.  Async on `stream`.  HIVE_EINVAL for null pointers with n > 0,
 * misalignment, or n_blocks outside [1, 2^32]. */
hive_status hive_gather_ceiling(const uint64_t* d_blocks, uint64_t n_blocks, const uint32_t* d_keys,
                                uint64_t n, uint32_t* d_out, void* stream);
/* The same gather with the read/write mix of an insert probe: mode 0 = read
 * only (as above); mode 1 = the group's leader then stores 8 B (s0 ^ 1) into
 * slot (key & 31) of the block; mode 2 = that slot is updated by a 64-bit CAS
 * (expected = the block's first word as read, new = that ^ 1; the CAS result
 * is folded into d_out).  d_blocks is written in modes 1-2.  HIVE_EINVAL for
 * mode > 2 or the conditions above. */
hive_status hive_gather_ceiling_rw(uint64_t* d_blocks, uint64_t n_blocks, const uint32_t* d_keys, uint64_t n,
                                   uint32_t* d_out, uint32_t mode, void* stream);

/* Split packed records (value << 32 | key) into key / value arrays. */
hive_status hive_unpack_kv(const uint64_t* d_kv, uint64_t n, uint32_t* d_keys,
                           uint32_t* d_vals, void* stream);

/* Human-readable text of a status / of the last CUDA error seen. */
const char* hive_status_string(hive_status s);
const char* hive_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HIVE_H */
