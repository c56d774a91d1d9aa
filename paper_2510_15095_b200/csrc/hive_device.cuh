// hive_device.cuh — device-side layout, hashing and warp-group primitives of the
// B200 Hive table (arXiv 2510.15095).  Header-only, included by hive_kernels.cu.
//
// Layout: the bucket array is one virtually
// contiguous range of n_b buckets x 32 slots x 8 B (256 B per bucket, 256 B
// aligned), each slot the packed word (value << 32) | key with
// EMPTY = all ones (A-9).  There is no separate freeMask array: the WABC
// claim mask is the ballot of EMPTY slots over the bucket that Step 1 has
// already loaded (PAPER:291-292 with the claim RMW moved onto the slot word
// itself, one 64-bit CAS).
//
// Warp groups: one operation is served by a group of G lanes (G = 8 by
// default), each lane holding 32/G slots loaded with one 256-bit (G = 8) or
// 128-bit (G = 16) vector load, so a warp keeps 32/G independent bucket probes
// in flight (PAPER:304's one-lane-per-slot WCME is G = 32).
#pragma once
#include <cstdint>

namespace hive {

constexpr uint64_t EMPTY = ~0ull;
constexpr uint32_t INVALID_KEY = 0xFFFFFFFFu;
constexpr int SLOTS = 32;                 // S = 32 slots per bucket
constexpr uint32_t FULL = 0xFFFFFFFFu;
constexpr uint32_t DEDUP_SEED = 0x2545F491u;

// ---- packed word, PAPER:180-187 --------------------------------------------------
__device__ __forceinline__ uint64_t pack(uint32_t k, uint32_t v) {
    return ((uint64_t)v << 32) | (uint64_t)k;
}
__device__ __forceinline__ uint32_t key_of(uint64_t p) { return (uint32_t)p; }
__device__ __forceinline__ uint32_t val_of(uint64_t p) { return (uint32_t)(p >> 32); }

// ---- Listing 1, PAPER:229-249 (full 32-bit output, reduction in addr(), A-1) ----
__device__ __forceinline__ uint32_t bithash1(uint32_t key) {
    key = ~key + (key << 15);
    key ^= (key >> 12);
    key += (key << 2);
    key ^= (key >> 4);
    key *= 2057u;
    key ^= (key >> 16);
    return key;
}
__device__ __forceinline__ uint32_t bithash2(uint32_t key) {
    key = (key + 0x7ed55d16u) + (key << 12);
    key = (key ^ 0xc761c23cu) ^ (key >> 19);
    key = (key + 0x165667b1u) + (key << 5);
    key = (key + 0xd3a2646cu) ^ (key << 9);
    key = (key + 0xfd7046c5u) + (key << 3);
    key = (key ^ 0xb55a4f09u) ^ (key >> 16);
    return key;
}
// ---- lookup-based pair, §V-B (reading A-26) ----------------------
// "precomputed lookup tables stored in GPU constant memory": CRC-32/IEEE
// (reflected polynomial 0xEDB88320) and CRC-64/XZ (reflected ECMA-182,
// 0xC96C5795D7870F42), both init/xorout all-ones, over the 4 little-endian key
// bytes; the CRC-64 result is reduced to its low 32 bits.  The tables are
// filled by init_hash_tables() (hive_kernels.cu) — only that translation unit's
// copy is ever read.
// The tables live in global memory and are read through the read-only L1
// path (__ldg), not in __constant__ memory as in the paper's design: the 32
// lanes of a warp index a table at 32 different bytes, which the constant
// cache serves one address at a time, while L1 serves them as a few sector
// wavefronts.
static __device__ uint32_t c_crc32_tab[256];
static __device__ uint64_t c_crc64_tab[256];
__device__ __forceinline__ uint32_t crc32_key(uint32_t key) {
    uint32_t c = 0xFFFFFFFFu;
#pragma unroll
    for (int i = 0; i < 4; ++i) c = __ldg(&c_crc32_tab[(c ^ (key >> (8 * i))) & 0xFFu]) ^ (c >> 8);
    return ~c;
}
__device__ __forceinline__ uint32_t crc64_key(uint32_t key) {
    uint64_t c = ~0ull;
#pragma unroll
    for (int i = 0; i < 4; ++i)
        c = __ldg(reinterpret_cast<const unsigned long long*>(&c_crc64_tab[(c ^ (key >> (8 * i))) & 0xFFu])) ^ (c >> 8);
    return (uint32_t)~c;
}
enum HashKind : uint32_t { HASH_BITHASH = 0, HASH_CRC = 1 };

// MurmurHash3 finaliser: shard routing and the per-batch owner-election table
// (independent of BitHash1/2).
__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    return h;
}

// Three fingerprint bits of a key in its bucket's spill word (independent of
// BitHash1/2).
constexpr uint32_t SPILL_SEED = 0x3C6EF372u;
__device__ __forceinline__ uint64_t spill_fp(uint32_t k) {
    const uint32_t x = fmix32(k ^ SPILL_SEED);
    return (1ull << (x & 63)) | (1ull << ((x >> 6) & 63)) | (1ull << ((x >> 12) & 63));
}

// ---- device control block --------------------------------------------------------
struct Ctrl {
    unsigned long long count;          // live keys (buckets + stash), A-19
    unsigned long long stash_tail;     // ring slots used since the last drain
    unsigned long long n_left;         // Step-3 leftover list length (this phase)
    unsigned long long slow_next;      // Step-3 work queue cursor (this phase; cleared with n_left)
    unsigned long long evictions;      // Step-3 victim swaps
    unsigned long long max_depth;      // deepest Step-3 round count
    unsigned long long stash_pushes;   // Step-4 pushes
    unsigned long long leftovers;      // ops that reached Step 3
    unsigned long long failed;         // entries lost to a full stash (sticky)
    unsigned long long first_abort;    // merge: first aborting pair (LIFO index)
    unsigned long long dump_n;         // dump cursor
    unsigned long long in_b1;          // stats: keys resident in addr(h1)
    unsigned long long step3;          // entries placed by the Step-3 loop (cumulative)
    unsigned long long xfail;          // sharded: ops not sent (padded exchange region full), sticky
    unsigned long long eover;          // fused election: a part's table overflowed (sticky; never expected)
    unsigned long long cls_n[3];       // hive_mixed: ops per class (find, insert, erase) of the batch
    unsigned long long pad[1];
    // Algorithmic bytes touched, per kernel family: 256 per
    // bucket probe, 32 per CAS / atomic sector, 8 per spill word or stash word,
    // exact bytes of the key / value / result streams.
    unsigned long long abytes[8];
    // Insertion step breakdown (hive_profile level 2): warp
    // cycles spent in Step 1 (replace), Step 2 (claim-and-commit), Step 3
    // (bounded eviction) and Step 4 (stash fallback); per warp region,
    // max-over-lanes end minus min-over-lanes start of clock64().
    unsigned long long cyc[4];
};
enum AlgBytes { AB_FIND = 0, AB_INSERT = 1, AB_EVICT = 2, AB_ERASE = 3, AB_ELECT = 4, AB_RESIZE = 5 };

// ---- linear-hashing addressing, PAPER:485-503 (Litwin rule, A-2) ----------------
struct TableView {
    uint64_t* buckets;   // n_b * 32 packed words
    uint32_t mask;       // index_mask = 2^m - 1
    uint32_t split;      // split pointer
    // Spill filter (B200 addition): one 64-bit word per bucket b;
    // for every live key k NOT stored in bucket addr(h1(k)) (it sits in b2 or
    // the stash) the bits spill_fp(k) are set in spill[addr(h1(k))].  Bits are
    // only ever added (erase leaves them; split copies, merge ORs), so a word
    // missing any of k's bits proves k is in no place but b1.
    uint64_t* spill;
    uint32_t hkind;      // HashKind: the (h1, h2) pair of this table
    // The two hash functions: BitHash1/2 (Listing 1, default) or the lookup-
    // based CRC-32 / CRC-64 pair (§V-B).  The branch is warp-uniform.
    __device__ __forceinline__ uint32_t h1(uint32_t k) const {
        return hkind == HASH_CRC ? crc32_key(k) : bithash1(k);
    }
    __device__ __forceinline__ uint32_t h2(uint32_t k) const {
        return hkind == HASH_CRC ? crc64_key(k) : bithash2(k);
    }
    __device__ __forceinline__ uint32_t addr(uint32_t h) const {
        uint32_t b = h & mask;
        if (b < split) b = h & ((mask << 1) | 1u);
        return b;
    }
    // AltBucket (Alg. 3 line 34): the other candidate, equal -> cur,
    // neither -> first.
    __device__ __forceinline__ uint32_t alt(uint32_t k, uint32_t cur) const {
        uint32_t c1 = addr(h1(k)), c2 = addr(h2(k));
        return cur == c1 ? c2 : (cur == c2 ? c1 : c1);
    }
    __device__ __forceinline__ uint64_t* bucket(uint32_t b) const {
        return buckets + (uint64_t)b * SLOTS;
    }
};

// Overflow stash: a ring of packed words filled by fetch-add on
// tail, plus an open-addressing index key -> ring position so finds, erases
// and Step 1 can see stashed keys (A-10, A-11).
struct StashView {
    uint64_t* ring;      // cap words, EMPTY-initialised
    uint64_t* index;     // idx_mask + 1 words: (key << 32) | ring_pos, EMPTY = free
    uint64_t cap;
    uint64_t idx_mask;
    Ctrl* ctrl;
};

// Per-batch owner election table: (key << 32) | op, max op
// per key wins (= the oracle's last write).  `flag[op]` is set only for ops
// whose key occurs more than once in the phase, so only those consult the
// table again (uniform batches pay the election pass alone).
//
// For large phases the table is split into n_parts L2-sized sub-tables of
// mask + 1 entries; a key's sub-table is the top bits of its election hash and
// its home slot the low bits, so each per-part election launch works on an
// L2-resident sub-table.
struct DedupView {
    uint64_t* slots;     // nullptr = election disabled (HIVE_KEYS_UNIQUE)
    uint64_t mask;       // sub-table size - 1
    uint8_t* flag;       // per op (indexed like the keys), zeroed per phase
    uint32_t* owner_of;  // per op, written for flagged ops only
    uint32_t n_parts;    // sub-tables (power of two)
    uint8_t* any = nullptr;  // set to 1 by the election if it flags any op (zeroed with flag)
    __device__ __forceinline__ uint64_t* sub(uint32_t h) const {
        const uint32_t part = n_parts > 1 ? (uint32_t)(((uint64_t)h * n_parts) >> 32) : 0u;
        return slots + (uint64_t)part * (mask + 1);
    }
};

// A phase's duplicate fix-up (out[op] = out[owner_of[op]] for flagged ops)
// handed to the next phase's kernel of a mixed batch; flag == nullptr: none.
struct DupFix {
    const uint8_t* flag = nullptr;
    const uint32_t* owner_of = nullptr;
    const uint8_t* any = nullptr;   // nullable: the election's any-flag word
    uint8_t* out = nullptr;
    uint64_t n = 0;                 // ops of the batch (flags are indexed by op)
};

// ---- memory access -----------------------------------------------------------------
// Bucket loads: 256-bit vector loads (LDG.E.ENL2.256 on sm_100a), bypassing L1
// allocation (random, no reuse; also no stale L1 lines across the CAS traffic of
// other SMs).  A lane holding SPL slots issues SPL/4 of them back to back, so all
// of a probe's bytes are in flight at once.  `volatile` keeps re-probes of the
// same bucket (after a lost CAS) from being merged by the compiler.
__device__ __forceinline__ void ld4(const uint64_t* p, uint64_t& a, uint64_t& b, uint64_t& c,
                                    uint64_t& d) {
    asm volatile("ld.global.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}
// Read-only phase variant (FIND): the table is immutable for the whole kernel.
__device__ __forceinline__ void ld4_ro(const uint64_t* p, uint64_t& a, uint64_t& b, uint64_t& c,
                                       uint64_t& d) {
    asm("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
        : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}
template <int SPL>
__device__ __forceinline__ void load_slots(const uint64_t* p, uint64_t (&s)[SPL]) {
    if constexpr (SPL >= 4) {
#pragma unroll
        for (int i = 0; i < SPL; i += 4) ld4(p + i, s[i], s[i + 1], s[i + 2], s[i + 3]);
    } else if constexpr (SPL == 2) {
        asm volatile("ld.global.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(s[0]), "=l"(s[1]) : "l"(p));
    } else {
        asm volatile("ld.global.L1::no_allocate.u64 %0, [%1];" : "=l"(s[0]) : "l"(p));
    }
}
template <int SPL>
__device__ __forceinline__ void load_slots_ro(const uint64_t* p, uint64_t (&s)[SPL]) {
    if constexpr (SPL >= 4) {
#pragma unroll
        for (int i = 0; i < SPL; i += 4) ld4_ro(p + i, s[i], s[i + 1], s[i + 2], s[i + 3]);
    } else if constexpr (SPL == 2) {
        asm("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(s[0]), "=l"(s[1]) : "l"(p));
    } else {
        asm("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(s[0]) : "l"(p));
    }
}

// ---- warp-group view ---------------------------------------------------------------
template <int G>
struct WarpGroup {
    static constexpr int SPL = SLOTS / G;          // slots per lane
    static constexpr int GPW = 32 / G;             // groups per warp
    static constexpr uint32_t GMASK = (G == 32) ? FULL : ((1u << G) - 1u);
    int lane, gi, gl;
    __device__ __forceinline__ WarpGroup() {
        lane = threadIdx.x & 31;
        gi = lane / G;
        gl = lane % G;
    }
    __device__ __forceinline__ int base() const { return gi * G; }
    // this group's bits of a full-warp ballot
    __device__ __forceinline__ uint32_t bits(uint32_t bal) const {
        return (bal >> (gi * G)) & GMASK;
    }
    __device__ __forceinline__ uint32_t ballot(bool p) const {
        return bits(__ballot_sync(FULL, p));
    }
    template <typename T>
    __device__ __forceinline__ T bcast(T v, int src_gl) const {
        return __shfl_sync(FULL, v, base() + src_gl);
    }
    __device__ __forceinline__ uint64_t* slot_ptr(uint64_t* bucket) const {
        return bucket + gl * SPL;
    }
};

// Select s[j] for a runtime j without local-memory indexing.
template <int SPL>
__device__ __forceinline__ uint64_t pick(const uint64_t (&s)[SPL], int j) {
    uint64_t w = s[0];
#pragma unroll
    for (int i = 1; i < SPL; ++i)
        if (i == j) w = s[i];
    return w;
}
template <int SPL>
__device__ __forceinline__ void put(uint64_t (&s)[SPL], int j, uint64_t w) {
#pragma unroll
    for (int i = 0; i < SPL; ++i)
        if (i == j) s[i] = w;
}

// One pass over a lane's slots (WCME compare + WABC free test):
// jm = first slot holding key k, jf = first EMPTY slot (SPL = none).  A slot is
// EMPTY iff its key word is 0xFFFFFFFF (that key is reserved, A-9), so both
// tests are 32-bit compares; the scan runs high to low so the lowest index wins.
template <int SPL>
__device__ __forceinline__ void scan_slots(const uint64_t (&s)[SPL], uint32_t k, int& jm, int& jf) {
    jm = SPL;
    jf = SPL;
#pragma unroll
    for (int j = SPL - 1; j >= 0; --j) {
        const uint32_t key = key_of(s[j]);
        jm = (key == k) ? j : jm;
        jf = (key == INVALID_KEY) ? j : jf;
    }
}
// As scan_slots, but jf = the first EMPTY slot in cyclic order from `rot`
// (0 <= rot < SPL): concurrent claimers of one bucket start their free-slot
// search at different slots (placement is not observable).
template <int SPL>
__device__ __forceinline__ void scan_slots_rot(const uint64_t (&s)[SPL], uint32_t k, uint32_t rot, int& jm,
                                               int& jf) {
    jm = SPL;
    uint32_t fm = 0;
#pragma unroll
    for (int j = SPL - 1; j >= 0; --j) {
        const uint32_t key = key_of(s[j]);
        jm = (key == k) ? j : jm;
        fm |= (key == INVALID_KEY ? 1u : 0u) << j;
    }
    if (SPL == 1) {
        jf = fm ? 0 : SPL;
        return;
    }
    const uint32_t all = (1u << SPL) - 1u;
    const uint32_t r = ((fm >> rot) | (fm << (SPL - rot))) & all;
    jf = r ? (int)((__ffs(r) - 1 + rot) % SPL) : SPL;
}
// Lane `rot`-rotated first set bit of a G-bit group mask (-1 if none).
template <int G>
__device__ __forceinline__ int first_rot(uint32_t m, uint32_t rot) {
    if (G == 1) return m ? 0 : -1;
    constexpr uint32_t all = (G == 32) ? 0xFFFFFFFFu : ((1u << G) - 1u);
    const uint32_t r = rot ? (((m >> rot) | (m << (G - rot))) & all) : m;
    return r ? (int)((__ffs(r) - 1 + rot) % G) : -1;
}

// First slot holding k and its value (find path).
template <int SPL>
__device__ __forceinline__ int scan_value(const uint64_t (&s)[SPL], uint32_t k, uint32_t& v) {
    int jm = SPL;
#pragma unroll
    for (int j = SPL - 1; j >= 0; --j) {
        const bool hit = key_of(s[j]) == k;
        jm = hit ? j : jm;
        v = hit ? val_of(s[j]) : v;
    }
    return jm;
}

}  // namespace hive
