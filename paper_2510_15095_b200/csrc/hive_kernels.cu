// hive_kernels.cu — sm_100a kernels of the B200 Hive table (arXiv 2510.15095).
//
// Every kernel here is HBM-bound integer work (DESIGN.md "Kernels and their
// rooflines"): no tensor cores, no shared-memory tiling of the table (each
// 256 B bucket is touched once per probe).  Persistent grid-stride kernels of
// 256 threads; one operation per 8-lane group (4 slots = one 256-bit load per
// lane), so each warp keeps four independent bucket probes in flight.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "hive_kernels.cuh"

namespace hive {

// Claim placement inside a bucket (placement is not observable): 0 = the
// lowest free slot of the lowest lane with one (first-fit), 1 = a per-key
// rotated lane, 2 = rotated lane and slot.  Rotation cut lost optimistic
// claims (cfg2 leftovers 2.55 M -> 2.20 M) but made k_insert_fast slower
// (4.99 -> 5.37 ms, profiles/r02_claim_rot_sweep.jsonl): first-fit is kept.
constexpr uint32_t c_claim_rot = CLAIM_ROT_DEFAULT;

// --------------------------------------------------------------------------------
// small helpers
// --------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t cas64(uint64_t* p, uint64_t cmp, uint64_t val) {
    return (uint64_t)atomicCAS((unsigned long long*)p, (unsigned long long)cmp,
                               (unsigned long long)val);
}
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ unsigned long long warp_max(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long u = __shfl_xor_sync(FULL, v, o);
        v = u > v ? u : v;
    }
    return v;
}
__device__ __forceinline__ long long warp_min_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long u = __shfl_xor_sync(FULL, v, o);
        v = u < v ? u : v;
    }
    return v;
}
__device__ __forceinline__ long long warp_max_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long u = __shfl_xor_sync(FULL, v, o);
        v = u > v ? u : v;
    }
    return v;
}
// Warp-granularity region time: max over lanes of the end clock
// minus min over lanes of the start clock.
__device__ __forceinline__ unsigned long long warp_span(long long t_start, long long t_end) {
    return (unsigned long long)(warp_max_ll(t_end) - warp_min_ll(t_start));
}

// One global atomic per block for a per-thread counter.  Every thread of the
// block must call it (kernel epilogue, after the grid-stride loop).
__device__ __forceinline__ void block_add(unsigned long long* dst, unsigned long long v) {
    __shared__ unsigned long long acc;
    if (threadIdx.x == 0) acc = 0;
    __syncthreads();
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&acc, v);
    __syncthreads();
    if (threadIdx.x == 0 && acc) atomicAdd(dst, acc);
    __syncthreads();                       // acc is reused by the next call
}
__device__ __forceinline__ void block_max(unsigned long long* dst, unsigned long long v) {
    __shared__ unsigned long long accm;
    if (threadIdx.x == 0) accm = 0;
    __syncthreads();
    v = warp_max(v);
    if ((threadIdx.x & 31) == 0 && v) atomicMax(&accm, v);
    __syncthreads();
    if (threadIdx.x == 0 && accm) atomicMax(dst, accm);
    __syncthreads();
}

// Per-warp staging of an index list in shared memory; one global atomic per
// 32 items instead of one per warp-iteration.
struct WarpList {
    uint32_t* sbuf;   // 32 entries of this warp
    int n;            // warp-uniform fill level
    __device__ __forceinline__ void flush(uint32_t* out, unsigned long long* out_n) {
        __syncwarp();
        if (n == 0) return;
        const int lane = threadIdx.x & 31;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(out_n, (unsigned long long)n);
        base = __shfl_sync(FULL, base, 0);
        if (lane < n) out[base + lane] = sbuf[lane];
        __syncwarp();
        n = 0;
    }
    __device__ __forceinline__ void push(bool flag, uint32_t item, uint32_t* out,
                                         unsigned long long* out_n) {
        uint32_t bal = __ballot_sync(FULL, flag);
        int c = __popc(bal);
        if (c == 0) return;
        if (n + c > 32) flush(out, out_n);
        if (flag) sbuf[n + __popc(bal & lanemask_lt())] = item;
        n += c;
        __syncwarp();
    }
};

// --------------------------------------------------------------------------------
// stash index (reading A-10): open addressing on fmix32(key)
// --------------------------------------------------------------------------------
__device__ __forceinline__ void stash_index_put(const StashView& sv, uint32_t k, uint64_t pos) {
    uint64_t h = fmix32(k) & sv.idx_mask;
    const uint64_t w = ((uint64_t)k << 32) | pos;
    for (uint64_t probe = 0; probe <= sv.idx_mask; ++probe) {
        uint64_t e = sv.index[h];
        if (e == EMPTY) {
            uint64_t prev = cas64(&sv.index[h], EMPTY, w);
            if (prev == EMPTY) return;
            e = prev;
        }
        if ((uint32_t)(e >> 32) == k) {          // re-point a stale entry for k
            atomicExch((unsigned long long*)&sv.index[h], (unsigned long long)w);
            return;
        }
        h = (h + 1) & sv.idx_mask;
    }
}
// Ring position of the live stash entry holding k, or -1.
__device__ __forceinline__ int64_t stash_lookup(const StashView& sv, uint32_t k, uint64_t* word) {
    uint64_t h = fmix32(k) & sv.idx_mask;
    for (uint64_t probe = 0; probe <= sv.idx_mask; ++probe) {
        uint64_t e = sv.index[h];
        if (e == EMPTY) return -1;
        if ((uint32_t)(e >> 32) == k) {
            uint64_t pos = e & 0xFFFFFFFFull;
            uint64_t w = *(volatile uint64_t*)&sv.ring[pos];
            if (w != EMPTY && key_of(w) == k) {
                *word = w;
                return (int64_t)pos;
            }
            return -1;
        }
        h = (h + 1) & sv.idx_mask;
    }
    return -1;
}

// --------------------------------------------------------------------------------
// group protocols
// --------------------------------------------------------------------------------
template <int SPL>
__device__ __forceinline__ void fill_empty(uint64_t (&s)[SPL]) {
#pragma unroll
    for (int j = 0; j < SPL; ++j) s[j] = EMPTY;
}

// Step 1 / Alg. 1 ReplacePath and Alg. 4's CAS-to-EMPTY
// (PAPER:448-475): WCME on the cached bucket view -- per-lane first match, a
// group ballot = match mask M, FirstSet(M) elects the winner lane, which CASes
// its cached word to `newkv`; the outcome is broadcast by ballot.  On a lost CAS
// the winner refreshes its view and the group re-elects (reading A-18).
// Group-uniform result; all lanes call.
template <int G>
__device__ __forceinline__ bool wcme_cas(const WarpGroup<G>& wg, uint64_t (&s)[WarpGroup<G>::SPL],
                                         uint64_t* bucket, uint32_t k, uint64_t newkv,
                                         bool valid, uint32_t& ab) {
    constexpr int SPL = WarpGroup<G>::SPL;
    bool trying = valid, done = false;
    for (int iter = 0; iter <= SLOTS; ++iter) {
        int jm = SPL, jf;
        if (trying) scan_slots<SPL>(s, k, jm, jf);
        const uint32_t M = wg.ballot(jm < SPL);                   // match mask
        trying = trying && M != 0;                                // early exit
        if (!__any_sync(FULL, trying)) break;
        bool ok = false;
        if (trying && wg.gl == __ffs(M) - 1) {                    // FirstSet winner
            const uint64_t old = pick<SPL>(s, jm);
            const uint64_t prev = cas64(wg.slot_ptr(bucket) + jm, old, newkv);
            ab += 32;
            ok = (prev == old);
            if (!ok) put<SPL>(s, jm, prev);
        }
        const bool any_ok = wg.ballot(ok) != 0;                   // broadcast (all lanes)
        if (trying && any_ok) {
            done = true;
            trying = false;
        }
    }
    return done;
}

// Step 2 / WABC claim-and-commit: the ballot of EMPTY
// slots in the cached view is the claim mask; the lowest free lane elects its
// lowest free slot and publishes kv with ONE 64-bit CAS(EMPTY -> kv).  A lost
// CAS marks that slot taken in the view and the group re-elects.
template <int G>
__device__ __forceinline__ bool wabc_claim(const WarpGroup<G>& wg, uint64_t (&s)[WarpGroup<G>::SPL],
                                           uint64_t* bucket, uint64_t kv, bool want,
                                           uint32_t& ab) {
    constexpr int SPL = WarpGroup<G>::SPL;
    bool trying = want, placed = false;
    for (int iter = 0; iter <= SLOTS; ++iter) {
        int jm, jf = SPL;
        if (trying) scan_slots<SPL>(s, INVALID_KEY, jm, jf);
        const uint32_t F = wg.ballot(jf < SPL);
        trying = trying && F != 0;
        if (!__any_sync(FULL, trying)) break;
        bool ok = false;
        if (trying && wg.gl == __ffs(F) - 1) {
            const uint64_t prev = cas64(wg.slot_ptr(bucket) + jf, EMPTY, kv);
            ab += 32;
            ok = (prev == EMPTY);
            if (!ok) put<SPL>(s, jf, prev);
        }
        const bool any_ok = wg.ballot(ok) != 0;                   // all lanes vote
        if (trying && any_ok) {
            placed = true;
            trying = false;
        }
    }
    return placed;
}

// Optimistic WABC claim for the insert fast path: the lowest free lane (jf =
// its first free slot, from the Step-1 scan) issues CAS(EMPTY -> kv) but the
// group does NOT wait for the outcome; the CAS result is checked one loop
// iteration later (after the next op's loads are in flight) and a lost claim
// is handed to Step 3.  Returns group-uniformly whether a claim was issued.
template <int G>
__device__ __forceinline__ bool wabc_claim_issue(const WarpGroup<G>& wg, int jf, uint64_t* bucket, uint64_t kv,
                                                 bool want, bool& pend, uint64_t& pend_prev,
                                                 uint32_t& pend_item, uint32_t item, uint32_t& ab,
                                                 uint32_t lrot = 0) {
    constexpr int SPL = WarpGroup<G>::SPL;
    const uint32_t F = wg.ballot(want && jf < SPL);
    // the claiming lane is the first lane with a free slot in cyclic order
    // from a per-key rotation, so concurrent claimers of one bucket rarely
    // race for the same slot (a lost claim costs a Step-3 round)
    if (want && F && wg.gl == (lrot ? first_rot<G>(F, lrot) : __ffs(F) - 1)) {
        pend_prev = cas64(wg.slot_ptr(bucket) + jf, EMPTY, kv);
        pend = true;
        pend_item = item;
        ab += 32;
    }
    return want && F != 0;
}

// Read-only WCME for FIND: the value of the lowest matching slot (one 32-bit
// shuffle from the elected lane).
template <int G>
__device__ __forceinline__ bool wcme_value(const WarpGroup<G>& wg, const uint64_t (&s)[WarpGroup<G>::SPL],
                                           uint32_t k, bool valid, uint32_t* val) {
    constexpr int SPL = WarpGroup<G>::SPL;
    uint32_t mine = 0;
    const int jm = valid ? scan_value<SPL>(s, k, mine) : SPL;
    const uint32_t M = wg.ballot(jm < SPL);
    const uint32_t v = wg.bcast(mine, M ? __ffs(M) - 1 : 0);
    if (M) *val = v;
    return M != 0;
}

// Duplicate fix-up body (k_dup_copy's dense form; see there).
__device__ __forceinline__ void dup_fix(const DupFix& fx) {
    if (fx.any && *fx.any == 0) return;     // the election flagged nothing
    const uint64_t n = fx.n, nv = n / 16;
    const uint4* f4 = reinterpret_cast<const uint4*>(fx.flag);
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 w = f4[v];
        if ((w.x | w.y | w.z | w.w) == 0) continue;
        for (int j = 0; j < 16; ++j) {
            const uint64_t op = v * 16 + j;
            if (!fx.flag[op]) continue;
            const uint32_t o = fx.owner_of[op];
            if (o != (uint32_t)op) fx.out[op] = fx.out[o];
        }
    }
    for (uint64_t op = nv * 16 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; op < n;
         op += (uint64_t)gridDim.x * blockDim.x) {
        if (!fx.flag[op]) continue;
        const uint32_t o = fx.owner_of[op];
        if (o != (uint32_t)op) fx.out[op] = fx.out[o];
    }
}
// --------------------------------------------------------------------------------
// FIND: WCME on b1, then b2 only on a miss, then the stash
// index only when the stash is non-empty.  Read-only phase.
// --------------------------------------------------------------------------------
template <int G, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB)
k_find(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ idx, uint64_t n,
       const uint64_t* __restrict__ n_dev, TableView tv, StashView sv,
       uint32_t* __restrict__ vals_out, uint8_t* __restrict__ found_out, DupFix fx) {
    using WG = WarpGroup<G>;
    constexpr int SPL = WG::SPL;
    WG wg;
    if (fx.flag) dup_fix(fx);               // the ERASE phase's duplicate fix-up (mixed batch)
    if (n_dev) n = *n_dev;
    const bool stash_on = sv.ctrl->stash_tail != 0;
    uint32_t ab = 0;                       // per-thread: < 2^32 bytes
    const uint64_t warp = ((uint64_t)blockIdx.x * BLOCK + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * BLOCK) >> 5;
    // software pipeline: next iteration's (op, key) loads while this one probes
    const uint64_t stride = nw * WG::GPW;
    uint32_t op_n = 0, k_n = INVALID_KEY;
    {
        const uint64_t t = warp * WG::GPW + wg.gi;
        if (t < n) {
            op_n = idx ? idx[t] : (uint32_t)t;
            k_n = keys[op_n];
        }
    }
    for (uint64_t t0 = warp * WG::GPW; t0 < n; t0 += stride) {
        const uint64_t t = t0 + wg.gi;
        const bool active = t < n;
        const uint32_t op = op_n;                      // < 2^32 (API)
        const uint32_t k = active ? k_n : INVALID_KEY;
        if (t + stride < n) {
            op_n = idx ? idx[t + stride] : (uint32_t)(t + stride);
            k_n = keys[op_n];
        }
        const bool valid = k != INVALID_KEY;
        uint32_t b1 = 0, b2 = 0;
        if (valid) {
            b1 = tv.addr(tv.h1(k));
            b2 = tv.addr(tv.h2(k));
        }
        uint64_t s[SPL];
        uint64_t spill_w = 0;
        if (valid) {
            load_slots_ro<SPL>(wg.slot_ptr(tv.bucket(b1)), s);
            spill_w = __ldg((const unsigned long long*)&tv.spill[b1]);
        } else {
            fill_empty<SPL>(s);
        }
        uint32_t val = 0;
        bool found = wcme_value<G>(wg, s, k, valid, &val);
        // beyond b1 only if b1's spill word allows k to live elsewhere
        const bool maybe = valid && !found && (spill_w & spill_fp(k)) == spill_fp(k);
        const bool need2 = maybe && b2 != b1;
        if (__any_sync(FULL, need2)) {
            if (need2) load_slots_ro<SPL>(wg.slot_ptr(tv.bucket(b2)), s);
            found |= wcme_value<G>(wg, s, k, need2, &val);
        }
        if (stash_on && maybe && !found && wg.gl == 0) {
            uint64_t sw;
            if (stash_lookup(sv, k, &sw) >= 0) {
                found = true;
                val = val_of(sw);
            }
            ab += 16;
        }
        if (active && wg.gl == 0)
            ab += 8 + (found_out ? 1 : 0) + (valid ? 256 + 8 : 0) + (need2 ? 256 : 0);
        if (active && wg.gl == 0) {
            vals_out[op] = found ? val : 0u;
            if (found_out) found_out[op] = found ? 1 : 0;
        }
    }
    block_add(&sv.ctrl->abytes[AB_FIND], ab);
}

// --------------------------------------------------------------------------------
// Owner election for in-batch duplicates (reading A-15):
// insert-if-absent of (key << 32 | op) into a per-batch table; atomicMax keeps
// the highest op per key (the oracle's last write).  Lanes of a warp holding
// the same key elect their highest op first (op lists are in no particular
// order).  Every op whose key occurs more than once gets flag[op] = 1 (the
// first conflicting arrival flags the creator), so the phase kernels consult
// the table only for those ops; *dd.any = 1 once any op is flagged.
// --------------------------------------------------------------------------------
__device__ __forceinline__ void mark_any(const DedupView& dd, bool flagged) {
    if (__syncthreads_or(flagged) && threadIdx.x == 0 && dd.any) *dd.any = 1;
}
__global__ void __launch_bounds__(BLOCK)
k_dedup_elect(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ idx, uint64_t n,
              const uint64_t* __restrict__ n_dev, DedupView dd, Ctrl* ctrl,
              const uint32_t* __restrict__ idx2, const uint64_t* __restrict__ n_dev2, DedupView dd2) {
    // job 1: the ops of idx (or 0..n-1) into dd; job 2 (idx2 != nullptr, a
    // mixed batch's ERASE list next to its INSERT list): the ops of idx2 into
    // dd2, starting at a warp-aligned virtual index so no warp mixes the jobs
    if (n_dev) n = *n_dev;
    const uint64_t n2 = idx2 ? *n_dev2 : 0;
    const uint64_t ra = (n + 31) & ~31ull;
    uint32_t ab = 0;                       // per-thread: < 2^32 bytes
    bool flagged = false, flagged2 = false;
    const int lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * BLOCK;
    for (uint64_t v0 = (uint64_t)blockIdx.x * BLOCK + (threadIdx.x & ~31u); v0 < ra + n2; v0 += stride) {
        const bool second = v0 >= ra;                               // warp-uniform
        const DedupView& d = second ? dd2 : dd;
        const uint64_t t = (second ? v0 - ra : v0) + lane;
        const bool active = t < (second ? n2 : n);
        const uint32_t* li = second ? idx2 : idx;
        const uint32_t op = active ? (li ? li[t] : (uint32_t)t) : 0u;    // < 2^32 (API)
        const uint32_t k = active ? keys[op] : INVALID_KEY;
        const uint32_t grp = __match_any_sync(FULL, k);
        if (active) ab += 4 + (li ? 4 : 0);
        if (k == INVALID_KEY) continue;
        bool fl = false;
        uint32_t mx = op;
        if (__popc(grp) > 1) {
            d.flag[op] = 1;
            fl = true;
            mx = __reduce_max_sync(grp, op);
        }
        if (op == mx) {
            const uint64_t word = ((uint64_t)k << 32) | op;
            const uint32_t hk = fmix32(k ^ DEDUP_SEED);
            uint64_t* tab = d.sub(hk);
            uint64_t h = hk & d.mask;
            uint64_t probe = 0;
            for (; probe <= d.mask; ++probe) {
                const uint64_t prev = cas64(&tab[h], EMPTY, word);
                ab += 32;
                if (prev == EMPTY) break;
                if ((uint32_t)(prev >> 32) == k) {
                    d.flag[op] = 1;
                    d.flag[(uint32_t)prev] = 1;
                    fl = true;
                    if (word > prev) atomicMax((unsigned long long*)&tab[h], (unsigned long long)word);
                    break;
                }
                h = (h + 1) & d.mask;
            }
            if (probe > d.mask) atomicAdd(&ctrl->eover, 1ull);   // table full: never at the sizing (stats)
        }
        if (second) flagged2 |= fl;
        else flagged |= fl;
    }
    block_add(&ctrl->abytes[AB_ELECT], ab);
    mark_any(dd, flagged);
    if (idx2) mark_any(dd2, flagged2);
}

// Election over one part of a hash-partitioned phase: input = the part's
// (op << 32 | key) records in op order (stable partition), sub-table L2-resident.
__global__ void __launch_bounds__(BLOCK)
k_dedup_elect_part(const uint64_t* __restrict__ recs, const uint64_t* __restrict__ part_info, uint32_t part,
                   DedupView dd, Ctrl* ctrl, uint4* __restrict__ clear_next, uint64_t clear_n16) {
    const uint64_t n = part_info[part];
    const uint64_t base = part_info[MAX_PARTS + part];
    const int lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * BLOCK;
    uint32_t ab = 0;                       // per-thread: < 2^32 bytes
    bool flagged = false;
    for (uint64_t t0 = (uint64_t)blockIdx.x * BLOCK + (threadIdx.x & ~31u); t0 < n; t0 += stride) {
        const uint64_t t = t0 + lane;
        const bool active = t < n;
        const uint64_t w = active ? recs[base + t] : EMPTY;
        const uint32_t k = (uint32_t)w, op = (uint32_t)(w >> 32);
        const uint32_t grp = __match_any_sync(FULL, k);
        if (active) ab += 8;
        if (!active) continue;
        // input order inside a warp is arbitrary here: elect the max op of the
        // lanes holding the same key
        uint32_t mx = op;
        if (__popc(grp) > 1) {
            dd.flag[op] = 1;
            flagged = true;
            mx = __reduce_max_sync(grp, op);
        }
        if (op != mx) continue;
        const uint64_t word = ((uint64_t)k << 32) | op;
        const uint32_t hk = fmix32(k ^ DEDUP_SEED);
        uint64_t* tab = dd.sub(hk);
        uint64_t h = hk & dd.mask;
        uint64_t probe = 0;
        for (; probe <= dd.mask; ++probe) {
            const uint64_t prev = cas64(&tab[h], EMPTY, word);
            ab += 32;
            if (prev == EMPTY) break;
            if ((uint32_t)(prev >> 32) == k) {
                dd.flag[op] = 1;
                dd.flag[(uint32_t)prev] = 1;
                flagged = true;
                if (word > prev) atomicMax((unsigned long long*)&tab[h], (unsigned long long)word);
                break;
            }
            h = (h + 1) & dd.mask;
        }
        if (probe > dd.mask) atomicAdd(&ctrl->eover, 1ull);   // table full: never at the sizing (stats)
    }
    block_add(&ctrl->abytes[AB_ELECT], ab);
    // clear the NEXT part's sub-table (EMPTY = all ones) in this launch's
    // tail: the election is L2-atomic bound, so the writes use idle HBM time
    // and leave the next table's lines in L2 for its launch
    if (clear_next) {
        const uint4 e = make_uint4(~0u, ~0u, ~0u, ~0u);
        for (uint64_t i = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; i < clear_n16; i += stride) clear_next[i] = e;
    }
    mark_any(dd, flagged);
}

// The same election with two independent records per lane per iteration:
// both first CASes are issued back to back, so each lane keeps two L2 atomic
// round trips in flight (the one-record kernel is CAS-latency bound: 97% warps
// active, 64 long-scoreboard stalls per issue).  Collisions fall back to the
// sequential probe loop of their record.
__device__ __forceinline__ void elect_resolve(const DedupView& dd, uint64_t* tab, uint64_t h, uint64_t prev,
                                              uint64_t word, uint32_t k, uint32_t op, uint32_t& ab, Ctrl* ctrl) {
    for (uint64_t probe = 0;; ) {
        if (prev == EMPTY) return;
        if ((uint32_t)(prev >> 32) == k) {
            dd.flag[op] = 1;
            dd.flag[(uint32_t)prev] = 1;
            if (dd.any) *dd.any = 1;                         // rare: a duplicate across warps
            if (word > prev) atomicMax((unsigned long long*)&tab[h], (unsigned long long)word);
            return;
        }
        if (++probe > dd.mask) { atomicAdd(&ctrl->eover, 1ull); return; }
        h = (h + 1) & dd.mask;
        prev = cas64(&tab[h], EMPTY, word);
        ab += 32;
    }
}
template <int MINB>
__global__ void __launch_bounds__(BLOCK, MINB)
k_dedup_elect_part2(const uint64_t* __restrict__ recs, const uint64_t* __restrict__ part_info, uint32_t part,
                    DedupView dd, Ctrl* ctrl) {
    const uint64_t n = part_info[part];
    const uint64_t base = part_info[MAX_PARTS + part];
    const int lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * BLOCK * 2;
    uint32_t ab = 0;
    for (uint64_t t0 = ((uint64_t)blockIdx.x * BLOCK + (threadIdx.x & ~31u)) * 2; t0 < n; t0 += stride) {
        const uint64_t ta = t0 + lane, tb = t0 + 32 + lane;
        const uint64_t wa = ta < n ? recs[base + ta] : EMPTY;
        const uint64_t wb = tb < n ? recs[base + tb] : EMPTY;
        const uint32_t ka = (uint32_t)wa, opa = (uint32_t)(wa >> 32);
        const uint32_t kb = (uint32_t)wb, opb = (uint32_t)(wb >> 32);
        const uint32_t ga = __match_any_sync(FULL, ka), gb = __match_any_sync(FULL, kb);
        bool da = ta < n, db = tb < n;
        ab += (da ? 8 : 0) + (db ? 8 : 0);
        if (da && __popc(ga) > 1) {
            dd.flag[opa] = 1;
            if (dd.any) *dd.any = 1;
            da = __reduce_max_sync(ga, opa) == opa;
        } else if (__popc(ga) > 1) {
            (void)__reduce_max_sync(ga, opa);               // every lane of the group takes part
        }
        if (db && __popc(gb) > 1) {
            dd.flag[opb] = 1;
            if (dd.any) *dd.any = 1;
            db = __reduce_max_sync(gb, opb) == opb;
        } else if (__popc(gb) > 1) {
            (void)__reduce_max_sync(gb, opb);
        }
        const uint64_t worda = ((uint64_t)ka << 32) | opa, wordb = ((uint64_t)kb << 32) | opb;
        const uint32_t hka = fmix32(ka ^ DEDUP_SEED), hkb = fmix32(kb ^ DEDUP_SEED);
        uint64_t* taba = dd.sub(hka);
        uint64_t* tabb = dd.sub(hkb);
        const uint64_t ha = hka & dd.mask, hb = hkb & dd.mask;
        uint64_t pa = EMPTY, pb = EMPTY;
        if (da) { pa = cas64(&taba[ha], EMPTY, worda); ab += 32; }
        if (db) { pb = cas64(&tabb[hb], EMPTY, wordb); ab += 32; }
        if (da) elect_resolve(dd, taba, ha, pa, worda, ka, opa, ab, ctrl);
        if (db) elect_resolve(dd, tabb, hb, pb, wordb, kb, opb, ab, ctrl);
    }
    block_add(&ctrl->abytes[AB_ELECT], ab);
}

// Hash partition of one phase's ops for the election (order inside a part is
// arbitrary; the election is order-free): pass 1 per-block histograms,
// pass 2 per-part bases, pass 3 a 4096-op tile per block written part by part
// at a per-block reservation (runs of ~4096/P contiguous records).
constexpr int ETILE = 4096;
__device__ __forceinline__ uint32_t elect_part(uint32_t k, uint32_t n_parts) {
    return (uint32_t)(((uint64_t)fmix32(k ^ DEDUP_SEED) * (uint64_t)n_parts) >> 32);
}
// Warp-aggregated shared-memory count: one atomic per distinct part in the
// warp (lanes with part >= MAX_PARTS do not count); returns the lane's rank
// among the lanes of its part inside this warp's slice of the count.
// Lanes holding the same value of a 7-bit label, from 7 ballots (multisplit;
// MATCH.ANY measured ~3x slower here).
__device__ __forceinline__ uint32_t match7(uint32_t v) {
    uint32_t m = FULL;
#pragma unroll
    for (int b = 0; b < 7; ++b) {
        const uint32_t bal = __ballot_sync(FULL, (v >> b) & 1u);
        m &= ((v >> b) & 1u) ? bal : ~bal;
    }
    return m;
}
__device__ __forceinline__ uint32_t warp_part_add(unsigned int* hist, uint32_t part) {
    const uint32_t grp = match7(part);
    const int leader = __ffs(grp) - 1;
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (lane == leader && part < MAX_PARTS) base = atomicAdd(&hist[part], (unsigned)__popc(grp));
    base = __shfl_sync(FULL, base, leader);
    return base + __popc(grp & lanemask_lt());
}

__global__ void __launch_bounds__(BLOCK)
k_elect_hist(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ idx, uint64_t n,
             const uint64_t* __restrict__ n_dev, uint32_t n_parts, unsigned long long* __restrict__ gcount) {
    __shared__ unsigned int hist[MAX_PARTS];
    if (n_dev) n = *n_dev;
    for (int p = threadIdx.x; p < MAX_PARTS; p += BLOCK) hist[p] = 0;
    __syncthreads();
    constexpr int R = 4;                     // independent loads in flight per lane
    const uint64_t stride = (uint64_t)gridDim.x * BLOCK * R;
    for (uint64_t i0 = ((uint64_t)blockIdx.x * BLOCK + (threadIdx.x & ~31u)) * R; i0 < n; i0 += stride) {
        uint32_t k[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint64_t i = i0 + r * 32 + (threadIdx.x & 31);
            k[r] = i < n ? keys[idx ? idx[i] : i] : INVALID_KEY;
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (k[r] != INVALID_KEY) atomicAdd(&hist[elect_part(k[r], n_parts)], 1u);
    }
    __syncthreads();
    for (int p = threadIdx.x; p < (int)n_parts; p += BLOCK)
        if (hist[p]) atomicAdd(&gcount[p], (unsigned long long)hist[p]);
}
__global__ void k_elect_bases(const unsigned long long* __restrict__ gcount, uint32_t n_parts,
                              uint64_t* __restrict__ part_info, unsigned long long* __restrict__ cursor) {
    if (threadIdx.x != 0) return;
    uint64_t run = 0;
    for (uint32_t p = 0; p < n_parts; ++p) {
        part_info[p] = gcount[p];
        part_info[MAX_PARTS + p] = run;
        cursor[p] = run;
        run += gcount[p];
    }
}
// Tile of ETILE ops per block iteration: keys loaded first (PER per thread),
// warp-aggregated ranks in a shared histogram, the tile staged in shared
// memory grouped by part, one global reservation per (tile, part), then a
// coalesced copy-out (consecutive threads write consecutive records of a
// part's run).  Part and rank share one register (rank < 2^16, part < 2^7).
// WITH_VALS (the fused insert path): the op's value is staged and written
// beside its record (rvals, same order), and ops with the reserved key -- in
// no part -- get status 2 / value-out 0 here.
template <bool WITH_VALS>
__global__ void __launch_bounds__(BLOCK, 4)
k_elect_scatter(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ idx, uint64_t n,
                const uint64_t* __restrict__ n_dev, uint32_t n_parts, unsigned long long* __restrict__ cursor,
                uint64_t* __restrict__ recs, const uint32_t* __restrict__ vals, uint32_t* __restrict__ rvals,
                uint8_t* __restrict__ status, uint32_t* __restrict__ vals_zero) {
    __shared__ unsigned int hist[MAX_PARTS];
    __shared__ unsigned int loff[MAX_PARTS + 1];
    __shared__ unsigned long long gbase[MAX_PARTS];
    constexpr int TILE = WITH_VALS ? ETILE / 2 : ETILE;    // 48 KB static shared memory
    __shared__ uint64_t stage[TILE];
    __shared__ uint8_t stagep[TILE];                         // each staged record's part
    __shared__ uint32_t stagev[WITH_VALS ? TILE : 1];
    if (n_dev) n = *n_dev;
    constexpr int PER = TILE / BLOCK;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t t0 = (uint64_t)blockIdx.x * TILE; t0 < n; t0 += (uint64_t)gridDim.x * TILE) {
        for (int p = threadIdx.x; p < MAX_PARTS; p += BLOCK) hist[p] = 0;
        __syncthreads();
        // warp w owns elements [w * 32 * PER, (w + 1) * 32 * PER) of the tile
        const uint64_t wbase = t0 + (uint64_t)warp * 32 * PER + lane;
        uint32_t k[PER], pr[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const uint64_t i = wbase + (uint64_t)j * 32;
            k[j] = i < n ? keys[idx ? idx[i] : i] : INVALID_KEY;
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const uint32_t part = k[j] != INVALID_KEY ? elect_part(k[j], n_parts) : MAX_PARTS;
            const uint32_t rank = warp_part_add(hist, part);
            pr[j] = (part << 16) | rank;
        }
        __syncthreads();
        if (warp == 0) {                       // exclusive scan of the tile's part counts
            uint32_t run = 0;
            for (uint32_t p0 = 0; p0 < n_parts; p0 += 32) {
                const uint32_t p = p0 + lane;
                const uint32_t c = p < n_parts ? hist[p] : 0u;
                uint32_t x = c;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL, x, d);
                    if (lane >= d) x += y;
                }
                if (p < n_parts) {
                    loff[p] = run + x - c;
                    gbase[p] = c ? atomicAdd(&cursor[p], (unsigned long long)c) : 0ull;
                }
                run += __shfl_sync(FULL, x, 31);
            }
            if (lane == 0) loff[n_parts] = run;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const uint32_t part = pr[j] >> 16;
            const uint64_t i = wbase + (uint64_t)j * 32;
            if (part >= MAX_PARTS) {
                if (WITH_VALS && i < n) {                  // reserved key: in no part
                    const uint32_t op = idx ? idx[i] : (uint32_t)i;
                    if (status) status[op] = 2;
                    if (vals_zero) vals_zero[op] = 0;
                }
                continue;
            }
            const uint32_t op = idx ? idx[i] : (uint32_t)i;
            stage[loff[part] + (pr[j] & 0xFFFFu)] = ((uint64_t)op << 32) | k[j];
            stagep[loff[part] + (pr[j] & 0xFFFFu)] = (uint8_t)part;
            if constexpr (WITH_VALS) stagev[loff[part] + (pr[j] & 0xFFFFu)] = vals[op];
        }
        __syncthreads();
        const uint32_t total = loff[n_parts];
        for (uint32_t e = threadIdx.x; e < total; e += BLOCK) {
            const uint64_t rec = stage[e];
            const uint32_t part = stagep[e];
            recs[gbase[part] + (e - loff[part])] = rec;
            if constexpr (WITH_VALS) rvals[gbase[part] + (e - loff[part])] = stagev[e];
        }
        __syncthreads();
    }
}

cudaError_t launch_elect_partition(cudaStream_t s, const uint32_t* keys, const uint32_t* idx, uint64_t n,
                                   const uint64_t* n_dev, uint32_t n_parts, unsigned long long* gcount,
                                   unsigned long long* cursor, uint64_t* part_info, uint64_t* recs,
                                   int num_sms, const uint32_t* vals, uint32_t* rvals, uint8_t* status,
                                   uint32_t* vals_zero) {
    cudaError_t e = cudaMemsetAsync(gcount, 0, MAX_PARTS * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    const int grid_h = (int)std::min<uint64_t>((n + BLOCK - 1) / BLOCK, (uint64_t)num_sms * 8);
    k_elect_hist<<<grid_h, BLOCK, 0, s>>>(keys, idx, n, n_dev, n_parts, gcount);
    k_elect_bases<<<1, 32, 0, s>>>(gcount, n_parts, part_info, cursor);
    const int grid_s = (int)std::min<uint64_t>((n + ETILE - 1) / ETILE, (uint64_t)num_sms * 8);
    const int grid_v = (int)std::min<uint64_t>((n + ETILE / 2 - 1) / (ETILE / 2), (uint64_t)num_sms * 8);
    if (rvals)
        k_elect_scatter<true><<<grid_v, BLOCK, 0, s>>>(keys, idx, n, n_dev, n_parts, cursor, recs, vals, rvals,
                                                       status, vals_zero);
    else
        k_elect_scatter<false><<<grid_s, BLOCK, 0, s>>>(keys, idx, n, n_dev, n_parts, cursor, recs, nullptr,
                                                        nullptr, nullptr, nullptr);
    return cudaGetLastError();
}

__device__ __forceinline__ uint32_t dedup_owner(const DedupView& dd, uint32_t k, uint32_t self) {
    const uint32_t hk = fmix32(k ^ DEDUP_SEED);
    const uint64_t* tab = dd.sub(hk);
    uint64_t h = hk & dd.mask;
    for (uint64_t probe = 0; probe <= dd.mask; ++probe) {
        uint64_t e = tab[h];
        if (e == EMPTY) return self;
        if ((uint32_t)(e >> 32) == k) return (uint32_t)e;
        h = (h + 1) & dd.mask;
    }
    return self;
}

// Owner check of one group (all lanes call): only flagged ops probe the table.
template <int G>
__device__ __forceinline__ bool owns(const WarpGroup<G>& wg, const DedupView& dd, bool valid,
                                     uint32_t k, uint32_t op, uint32_t& ab) {
    if (!dd.slots) return true;
    uint32_t owner = (uint32_t)op;
    if (valid && wg.gl == 0) {
        ab += 1;
        if (dd.flag[op]) {
            owner = dedup_owner(dd, k, op);
            dd.owner_of[op] = owner;
            ab += 8 + 4;
        }
    }
    return wg.bcast(owner, 0) == op;
}

// --------------------------------------------------------------------------------
// INSERT fast path: Step 1 (replace) + Step 2 (claim-and-commit,
// PAPER:348-381) in one pass; ops whose candidate buckets are both full go to
// the leftover list for Steps 3-4.  The spill filter decides whether Step 1
// must look beyond b1; Step 2 reads b2 only when b1 is full.
//
// `kvs != nullptr` = place-only mode used to reinsert drained stash entries
// after a resize: Step 1 is skipped (those keys are in no bucket)
// and nothing is counted.
// --------------------------------------------------------------------------------
// Two-choice threshold test (signed, so a threshold of 0 compiles without a
// pointless-comparison warning).
__device__ __forceinline__ bool below_two_choice_t(uint32_t f) { return (int64_t)f < (int64_t)TWO_CHOICE_T; }

// EMPTY slots of the group's bucket view (all lanes of the group get the sum).
template <int G>
__device__ __forceinline__ uint32_t group_free(const uint64_t (&s)[WarpGroup<G>::SPL]) {
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < WarpGroup<G>::SPL; ++j) c += key_of(s[j]) == INVALID_KEY ? 1u : 0u;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) c += __shfl_xor_sync(FULL, c, o);
    return c;
}

// Per-thread state of the fast path that outlives one range of ops.
struct FastState {
    unsigned long long added = 0, cyc1 = 0, cyc2 = 0;
    uint32_t ab = 0;                       // per-thread: < 2^32 bytes
    bool pend = false;                     // this lane issued a claim last iteration
    uint64_t pend_prev = EMPTY;            // ... and this is its CAS result
    uint32_t pend_item = 0;
};

// The fast-path loop over the ops [lo, hi) of an op source, warp `warp` of
// `nw`: fetch(tt, op, k, v) reads op tt, owner(wg, valid, k, op, ab) is the
// group-uniform owner-election check.  in_bytes: streamed input / output bytes
// per op (byte accounting).  The claim issued by the last iteration is
// resolved before returning; the caller flushes `wl` and reduces `st`.
template <int G, bool PROF, class Fetch, class Owner>
__device__ __forceinline__ void insert_fast_range(uint64_t lo, uint64_t hi, uint64_t warp, uint64_t nw, Fetch fetch,
                                                  Owner owner, bool place_only, bool stash_on, uint32_t in_bytes,
                                                  TableView tv, StashView sv, uint8_t* __restrict__ status,
                                                  uint32_t* __restrict__ vals_zero, uint32_t* __restrict__ leftover,
                                                  WarpList& wl, FastState& st) {
    using WG = WarpGroup<G>;
    constexpr int SPL = WG::SPL;
    WG wg;
    // software pipeline: the next iteration's (op, key, value) is loaded while
    // this iteration probes
    const uint64_t stride = nw * WG::GPW;
    uint32_t op_n = 0, k_n = INVALID_KEY, v_n = 0;
    if (lo + warp * WG::GPW + wg.gi < hi) fetch(lo + warp * WG::GPW + wg.gi, op_n, k_n, v_n);
    for (uint64_t t0 = lo + warp * WG::GPW; t0 < hi; t0 += stride) {
        long long c0 = 0;
        if constexpr (PROF) c0 = clock64();
        const uint64_t t = t0 + wg.gi;
        const bool active = t < hi;
        const uint32_t op = op_n;                    // op indices < 2^32 (API contract)
        const uint32_t k = active ? k_n : INVALID_KEY;
        const uint32_t v = v_n;
        if (t + stride < hi) fetch(t + stride, op_n, k_n, v_n);
        bool valid = active && k != INVALID_KEY;
        uint32_t b1 = 0, b2 = 0, h2 = 0;
        if (valid) {
            b1 = tv.addr(tv.h1(k));
            h2 = tv.h2(k);
            b2 = tv.addr(h2);
        }
        // per-key start of the free-slot search (lane, slot): independent of b1
        // (c_claim_rot: 0 = lowest free, 1 = rotated lane, 2 = lane and slot)
        const uint32_t lrot = c_claim_rot >= 1 ? (h2 >> 24) % G : 0u;
        const uint32_t srot = c_claim_rot >= 2 ? (h2 >> 27) % WG::SPL : 0u;
        bool two = valid && b2 != b1;
        const uint64_t fp = spill_fp(k);
        // one bucket view: b1, later overwritten by b2 (b1's scan results are
        // kept in jm1 / jf1), so the two views never occupy registers together
        uint64_t sv_[SPL];
        uint64_t spill_w = 0;
        if (valid) {
            load_slots<SPL>(wg.slot_ptr(tv.bucket(b1)), sv_);
            spill_w = tv.spill[b1];
        } else {
            fill_empty<SPL>(sv_);
        }
        if (active && wg.gl == 0) {
            st.ab += in_bytes + (valid ? 256 + 8 : 0);
            if (!place_only) {
                if (vals_zero) vals_zero[op] = 0;
                if (!valid && status) status[op] = 2;
            }
        }
        // owner election: duplicates copy the owner's outcome afterwards
        if (!owner(wg, valid, k, op, st.ab)) {
            valid = false;
            two = false;
        }
        const uint64_t kv = pack(k, v);
        bool done = false, have2 = false;
        int jm1 = SPL, jf1 = SPL;
        [[maybe_unused]] uint32_t f1 = SPL * G;        // free slots of b1 (two-choice placement only)
        if (!place_only) {
            // Step 1: b1 (one scan gives the match and the first free slot); then
            // -- only if b1's spill word allows k to live elsewhere -- b2 and the
            // stash.
            if (valid) {
                if (c_claim_rot >= 2) scan_slots_rot<SPL>(sv_, k, srot, jm1, jf1);
                else scan_slots<SPL>(sv_, k, jm1, jf1);
            }
            if constexpr (TWO_CHOICE_T > 0) f1 = group_free<G>(sv_);
            if (__any_sync(FULL, wg.ballot(jm1 < SPL) != 0))
                done = wcme_cas<G>(wg, sv_, tv.bucket(b1), k, kv, valid, st.ab);
            const bool maybe = valid && !done && (spill_w & fp) == fp;
            const bool need2 = two && maybe;
            if (__any_sync(FULL, need2)) {
                if (need2) load_slots<SPL>(wg.slot_ptr(tv.bucket(b2)), sv_);
                if (need2 && wg.gl == 0) st.ab += 256;
                have2 = need2;
                done |= wcme_cas<G>(wg, sv_, tv.bucket(b2), k, kv, need2, st.ab);
            }
            if (stash_on) {
                bool sdone = false;
                if (maybe && !done && wg.gl == 0) {
                    uint64_t sw;
                    st.ab += 16;
                    int64_t pos = stash_lookup(sv, k, &sw);
                    while (pos >= 0) {
                        uint64_t prev = cas64(&sv.ring[pos], sw, kv);
                        if (prev == sw) { sdone = true; break; }
                        pos = stash_lookup(sv, k, &sw);
                    }
                }
                done |= wg.bcast(sdone, 0);
            }
        }
        long long c1 = 0;
        if constexpr (PROF) {
            c1 = clock64();
        }
        // resolve the claim issued in the previous iteration (its CAS has had
        // this iteration's loads to come back); a lost claim goes to Step 3
        wl.push(st.pend && st.pend_prev != EMPTY, st.pend_item, leftover, &sv.ctrl->n_left);
        st.pend = false;
        // Thresholded two-choice placement (reading A-21; placement is not
        // observable): when b1 has fewer than TWO_CHOICE_T free slots, b2 is
        // read and the emptier bucket is claimed.  TWO_CHOICE_T = 0: first-fit.
        bool choose2 = false;
        if constexpr (TWO_CHOICE_T > 0) {
            const bool look2 = !place_only && two && !done && below_two_choice_t(f1);
            if (__any_sync(FULL, look2)) {
                if (look2 && !have2) load_slots<SPL>(wg.slot_ptr(tv.bucket(b2)), sv_);
                if (look2 && !have2 && wg.gl == 0) st.ab += 256;
                if (look2) have2 = true;
                const uint32_t f2 = group_free<G>(sv_);
                choose2 = look2 && f2 > f1;
            }
        }
        // Step 2: optimistic WABC claim in b1, then b2 (first-fit, A-21); b2 is
        // read only if b1 is full.
        if (place_only && valid) {
            if (c_claim_rot >= 2) scan_slots_rot<SPL>(sv_, INVALID_KEY, srot, jm1, jf1);
            else scan_slots<SPL>(sv_, INVALID_KEY, jm1, jf1);
        }
        bool placed = wabc_claim_issue<G>(wg, jf1, tv.bucket(b1), kv, valid && !done && !choose2, st.pend,
                                          st.pend_prev, st.pend_item, op, st.ab, lrot);
        const bool want2 = two && !done && !placed;
        if (__any_sync(FULL, want2)) {
            if (want2 && !have2) load_slots<SPL>(wg.slot_ptr(tv.bucket(b2)), sv_);
            if (want2 && !have2 && wg.gl == 0) st.ab += 256;
            int jm2, jf2 = SPL;
            if (want2) {
                if (c_claim_rot >= 2) scan_slots_rot<SPL>(sv_, INVALID_KEY, srot, jm2, jf2);
                else scan_slots<SPL>(sv_, INVALID_KEY, jm2, jf2);
            }
            const bool p2 = wabc_claim_issue<G>(wg, jf2, tv.bucket(b2), kv, want2, st.pend, st.pend_prev,
                                                st.pend_item, op, st.ab, lrot);
            if (p2 && wg.gl == 0) {
                atomicOr((unsigned long long*)&tv.spill[b1], (unsigned long long)fp);
                st.ab += 8;
            }
            placed |= p2;
        }
        const bool left = valid && !done && !placed;
        if (!place_only && valid && wg.gl == 0) {
            if (status) status[op] = done ? 1 : 0;
            if (!done) ++st.added;
        }
        wl.push(left && wg.gl == 0, op, leftover, &sv.ctrl->n_left);
        if constexpr (PROF) {
            const long long c2 = clock64();
            const unsigned long long s1 = warp_span(c0, c1), s2 = warp_span(c1, c2);
            if (wg.lane == 0) {
                st.cyc1 += s1;
                st.cyc2 += s2;
            }
        }
    }
    wl.push(st.pend && st.pend_prev != EMPTY, st.pend_item, leftover, &sv.ctrl->n_left);
    st.pend = false;
}

// The standalone fast-path kernel keeps its own loop (the round-1 code): the
// same loop factored through insert_fast_range measured 7% slower here
// (5.13 vs 4.79 ms per cfg2 phase on one box, same DRAM bytes).
template <int G, int MINB, bool PROF = false>
__global__ void __launch_bounds__(BLOCK, MINB)
k_insert_fast(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
              const uint64_t* __restrict__ kvs, const uint32_t* __restrict__ idx, uint64_t n,
              const uint64_t* __restrict__ n_dev, TableView tv, StashView sv, DedupView dd,
              uint8_t* __restrict__ status, uint32_t* __restrict__ vals_zero,
              uint32_t* __restrict__ leftover, uint32_t op_base) {
    using WG = WarpGroup<G>;
    constexpr int SPL = WG::SPL;
    __shared__ uint32_t lbuf[WARPS_PER_BLOCK][32];
    WG wg;
    WarpList wl{lbuf[threadIdx.x >> 5], 0};
    if (n_dev) n = *n_dev;
    const bool place_only = kvs != nullptr;
    const bool stash_on = !place_only && sv.ctrl->stash_tail != 0;
    unsigned long long added = 0;
    uint32_t ab = 0;                       // per-thread: < 2^32 bytes
    bool pend = false;                     // this lane issued a claim last iteration
    uint64_t pend_prev = EMPTY;            // ... and this is its CAS result
    uint32_t pend_item = 0;
    const uint64_t warp = ((uint64_t)blockIdx.x * BLOCK + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * BLOCK) >> 5;
    // software pipeline: the next iteration's (op, key, value) is loaded while
    // this iteration probes
    const uint64_t stride = nw * WG::GPW;
    uint32_t op_n = 0, k_n = INVALID_KEY, v_n = 0;
    auto fetch = [&](uint64_t tt) {
        if (tt >= n) return;
        if (place_only) {
            const uint64_t w = kvs[tt];
            op_n = (uint32_t)tt;
            k_n = key_of(w);
            v_n = val_of(w);
        } else {
            op_n = idx ? idx[tt] : op_base + (uint32_t)tt;   // op_base: chunked launches
            k_n = keys[op_n];
            v_n = vals[op_n];
        }
    };
    fetch(warp * WG::GPW + wg.gi);
    unsigned long long cyc1 = 0, cyc2 = 0;   // PROF: this warp's Step-1 / Step-2 cycles
    for (uint64_t t0 = warp * WG::GPW; t0 < n; t0 += stride) {
        long long c0 = 0;
        if constexpr (PROF) c0 = clock64();
        const uint64_t t = t0 + wg.gi;
        const bool active = t < n;
        const uint32_t op = op_n;                    // op indices < 2^32 (API contract)
        const uint32_t k = active ? k_n : INVALID_KEY;
        const uint32_t v = v_n;
        fetch(t + stride);
        bool valid = active && k != INVALID_KEY;
        uint32_t b1 = 0, b2 = 0;
        if (valid) {
            b1 = tv.addr(tv.h1(k));
            b2 = tv.addr(tv.h2(k));
        }
        bool two = valid && b2 != b1;
        const uint64_t fp = spill_fp(k);
        // one bucket view: b1, later overwritten by b2 (b1's scan results are
        // kept in jm1 / jf1), so the two views never occupy registers together
        uint64_t sv_[SPL];
        uint64_t spill_w = 0;
        if (valid) {
            load_slots<SPL>(wg.slot_ptr(tv.bucket(b1)), sv_);
            spill_w = tv.spill[b1];
        } else {
            fill_empty<SPL>(sv_);
        }
        if (active && wg.gl == 0) {
            ab += (place_only ? 8 : 8 + (status ? 1 : 0) + (vals_zero ? 4 : 0) + (idx ? 4 : 0)) +
                  (valid ? 256 + 8 : 0);
            if (!place_only) {
                if (vals_zero) vals_zero[op] = 0;
                if (!valid && status) status[op] = 2;
            }
        }
        // owner election: duplicates copy the owner's outcome afterwards
        if (!owns<G>(wg, dd, valid, k, op, ab)) {
            valid = false;
            two = false;
        }
        const uint64_t kv = pack(k, v);
        bool done = false, have2 = false;
        int jm1 = SPL, jf1 = SPL;
        [[maybe_unused]] uint32_t f1 = SPL * G;        // free slots of b1 (two-choice placement only)
        if (!place_only) {
            // Step 1: b1 (one scan gives the match and the first free slot); then
            // -- only if b1's spill word allows k to live elsewhere -- b2 and the
            // stash.
            if (valid) scan_slots<SPL>(sv_, k, jm1, jf1);
            if constexpr (TWO_CHOICE_T > 0) f1 = group_free<G>(sv_);
            if (__any_sync(FULL, wg.ballot(jm1 < SPL) != 0))
                done = wcme_cas<G>(wg, sv_, tv.bucket(b1), k, kv, valid, ab);
            const bool maybe = valid && !done && (spill_w & fp) == fp;
            const bool need2 = two && maybe;
            if (__any_sync(FULL, need2)) {
                if (need2) load_slots<SPL>(wg.slot_ptr(tv.bucket(b2)), sv_);
                if (need2 && wg.gl == 0) ab += 256;
                have2 = need2;
                done |= wcme_cas<G>(wg, sv_, tv.bucket(b2), k, kv, need2, ab);
            }
            if (stash_on) {
                bool sdone = false;
                if (maybe && !done && wg.gl == 0) {
                    uint64_t sw;
                    ab += 16;
                    int64_t pos = stash_lookup(sv, k, &sw);
                    while (pos >= 0) {
                        uint64_t prev = cas64(&sv.ring[pos], sw, kv);
                        if (prev == sw) { sdone = true; break; }
                        pos = stash_lookup(sv, k, &sw);
                    }
                }
                done |= wg.bcast(sdone, 0);
            }
        }
        long long c1 = 0;
        if constexpr (PROF) c1 = clock64();
        // resolve the claim issued in the previous iteration (its CAS has had
        // this iteration's loads to come back); a lost claim goes to Step 3
        wl.push(pend && pend_prev != EMPTY, pend_item, leftover, &sv.ctrl->n_left);
        pend = false;
        // Thresholded two-choice placement (reading A-21; build-time, off by
        // default -- measured, §5): below TWO_CHOICE_T free slots in b1, read b2
        // and claim the emptier bucket.
        bool choose2 = false;
        if constexpr (TWO_CHOICE_T > 0) {
            const bool look2 = !place_only && two && !done && below_two_choice_t(f1);
            if (__any_sync(FULL, look2)) {
                if (look2 && !have2) load_slots<SPL>(wg.slot_ptr(tv.bucket(b2)), sv_);
                if (look2 && !have2 && wg.gl == 0) ab += 256;
                if (look2) have2 = true;
                const uint32_t f2 = group_free<G>(sv_);
                choose2 = look2 && f2 > f1;
            }
        }
        // Step 2: optimistic WABC claim in b1, then b2 (first-fit, A-21); b2 is
        // read only if b1 is full.
        if (place_only && valid) scan_slots<SPL>(sv_, INVALID_KEY, jm1, jf1);
        bool placed = wabc_claim_issue<G>(wg, jf1, tv.bucket(b1), kv, valid && !done && !choose2, pend, pend_prev,
                                          pend_item, op, ab);
        const bool want2 = two && !done && !placed;
        if (__any_sync(FULL, want2)) {
            if (want2 && !have2) load_slots<SPL>(wg.slot_ptr(tv.bucket(b2)), sv_);
            if (want2 && !have2 && wg.gl == 0) ab += 256;
            int jm2, jf2 = SPL;
            if (want2) scan_slots<SPL>(sv_, INVALID_KEY, jm2, jf2);
            const bool p2 = wabc_claim_issue<G>(wg, jf2, tv.bucket(b2), kv, want2, pend, pend_prev,
                                                pend_item, op, ab);
            if (p2 && wg.gl == 0) {
                atomicOr((unsigned long long*)&tv.spill[b1], (unsigned long long)fp);
                ab += 8;
            }
            placed |= p2;
        }
        const bool left = valid && !done && !placed;
        if (!place_only && valid && wg.gl == 0) {
            if (status) status[op] = done ? 1 : 0;
            if (!done) ++added;
        }
        wl.push(left && wg.gl == 0, op, leftover, &sv.ctrl->n_left);
        if constexpr (PROF) {
            const long long c2 = clock64();
            const unsigned long long s1 = warp_span(c0, c1), s2 = warp_span(c1, c2);
            if (wg.lane == 0) {
                cyc1 += s1;
                cyc2 += s2;
            }
        }
    }
    wl.push(pend && pend_prev != EMPTY, pend_item, leftover, &sv.ctrl->n_left);
    wl.flush(leftover, &sv.ctrl->n_left);
    block_add(&sv.ctrl->count, added);
    block_add(&sv.ctrl->abytes[AB_INSERT], ab);
    if constexpr (PROF) {
        block_add(&sv.ctrl->cyc[0], cyc1);
        block_add(&sv.ctrl->cyc[1], cyc2);
    }

}


// --------------------------------------------------------------------------------
// INSERT slow path: Step 3 bounded cuckoo eviction (Alg. 3)
// then Step 4 stash for the leftovers of the fast pass.
// B200 variant: no bucket lock -- the victim is swapped out with
// one 64-bit CAS(victim -> newcomer) (reading A-14) and the victim slot
// rotates with the round (reading A-6 allows any victim rule; placement is not
// observable).
// --------------------------------------------------------------------------------
// The Step 3-4 work loop as a device function: k_insert_slow runs it alone,
// the monolithic mixed kernel (k_mixed_mono) runs it as its eviction stage.
// Every thread of the grid must call it (block-level counter reductions).
template <int G, bool PROF>
__device__ __forceinline__ void insert_slow_body(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                                                 const uint64_t* __restrict__ kvs,
                                                 const uint32_t* __restrict__ leftover, TableView tv, StashView sv,
                                                 uint32_t max_evictions, uint8_t* __restrict__ status) {
    using WG = WarpGroup<G>;
    constexpr int SPL = WG::SPL;
    WG wg;
    const uint64_t n = sv.ctrl->n_left;
    if (!kvs && blockIdx.x == 0 && threadIdx.x == 0 && n) atomicAdd(&sv.ctrl->leftovers, (unsigned long long)n);
    unsigned long long evict = 0, depth = 0, pushes = 0, lost = 0, st3 = 0;
    uint32_t ab = 0;                       // per-thread: < 2^32 bytes
    // Dynamic scheduling: every warp iteration advances each busy group by one
    // eviction round; a group whose entry is placed (or stashed) immediately
    // takes the next leftover, so a warp never idles behind its longest chain.
    // Jobs come from a warp buffer: lane l holds the item and entry of leftover
    // position base + l, claimed 32 at a time with one atomic and loaded ahead
    // (items at the claim, entries during the next round), so starting a job is
    // a shuffle, not a dependent atomic -> item -> key/value load chain.
    bool busy = false;                       // group-uniform job state
    uint32_t item = 0, b = 0, seed = 0, r = 0;
    uint64_t kv = EMPTY;
    const int lane = threadIdx.x & 31;
    uint32_t q_item = 0;                     // this lane's buffered job
    uint64_t q_kv = EMPTY;
    uint32_t qa = 0, qn = 0;                 // warp-uniform: next buffered job, buffered jobs
    bool kv_due = false;                     // warp-uniform: q_kv not loaded yet
    bool drained = n == 0;                   // warp-uniform: no positions left to claim
    auto refill = [&]() {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&sv.ctrl->slow_next, 32ull);
        base = __shfl_sync(FULL, base, 0);
        qa = 0;
        qn = base >= n ? 0u : (uint32_t)(n - base < 32 ? n - base : 32);
        if (base + 32 >= n) drained = true;
        if ((uint32_t)lane < qn) q_item = leftover[base + lane];
        kv_due = qn != 0;
    };
    auto load_kv = [&]() {
        if (kv_due && (uint32_t)lane < qn) q_kv = kvs ? kvs[q_item] : pack(keys[q_item], vals[q_item]);
        kv_due = false;
    };
    if (!drained) refill();
    bool have = false;                       // s already holds bucket b (prefetched)
    uint64_t s[SPL];
    const uint32_t leaders = __ballot_sync(FULL, wg.gl == 0);
    unsigned long long cyc3 = 0, cyc4 = 0;    // PROF: this warp's Step-3 / Step-4 cycles
    while (true) {
        long long c0 = 0;
        if constexpr (PROF) c0 = clock64();
        // ---- hand out work to idle groups ----
        const uint32_t idle = __ballot_sync(FULL, !busy && wg.gl == 0);
        if (drained && qa == qn && idle == leaders) break;
        if (idle && qa < qn) {
            load_kv();                                         // no-op unless the buffer is fresh
            const uint32_t need = __popc(idle);
            const uint32_t rank = wg.bcast((uint32_t)__popc(idle & lanemask_lt()), 0);
            const uint32_t take = need < qn - qa ? need : qn - qa;
            const bool start = !busy && rank < take;           // group-uniform
            const int src = (int)(qa + (start ? rank : 0u));
            const uint32_t it = __shfl_sync(FULL, q_item, src);
            const uint64_t e = __shfl_sync(FULL, q_kv, src);
            qa += take;
            if (start) {
                item = it;
                kv = e;
                b = tv.addr(tv.h1(key_of(kv)));               // start at b1
                seed = tv.h2(key_of(kv));
                r = 0;
                busy = true;
                have = false;
                if (wg.gl == 0) ab += 4 + 8;
            }
        }
        if (qa == qn && !drained) refill();
        if (!__any_sync(FULL, busy)) {
            load_kv();
            if constexpr (PROF) {
                const unsigned long long sp = warp_span(c0, clock64());
                if (lane == 0) cyc3 += sp;
            }
            continue;
        }
        // ---- one round of Alg. 3 for every busy group ----
        if (busy && !have) {
            load_slots<SPL>(wg.slot_ptr(tv.bucket(b)), s);
            if (wg.gl == 0) ab += 256;
        } else if (!busy) {
            fill_empty<SPL>(s);
        }
        have = false;
        load_kv();                                             // overlaps this round's bucket load
        const bool placed = wabc_claim<G>(wg, s, tv.bucket(b), kv, busy, ab);   // line 3
        if (placed) {
            const uint32_t hb = tv.addr(tv.h1(key_of(kv)));
            if (wg.gl == 0 && hb != b) {
                atomicOr((unsigned long long*)&tv.spill[hb], (unsigned long long)spill_fp(key_of(kv)));
                ab += 8;
            }
        }
        // Victim (lines 17-21): a rotating slot (reading A-6: any victim rule;
        // preferring residents in their second bucket raised p_h1 to 0.93 but
        // doubled evictions and grew the stash 5x -- a net loss).
        const bool evicting = busy && !placed;
        const int vrot = (int)((seed + r * 11u) & 31u);       // the rotating slot
        int vs = vrot;
        uint64_t victim;
        bool alt_known = false;                              // nb_alt holds the victim's other bucket
        uint32_t nb_alt = 0;
        // (not for the lookup-based CRC pair: on, it lifts CRC inserts
        // 8.15 -> 8.33 G/s but the extra branch costs the default BitHash
        // kernels ~0.5%, profiles/r02f_crc_victim_ab.txt)
        if (VICTIM_LOOK > 0 && tv.hkind != HASH_CRC) {
            // Split-aware victim (A-6 allows any rule; placement is not
            // observable): each lane offers NC candidates, its slots
            // o, o + ST, o + 2 ST, ... (ST = SPL / NC, o = the rotating slot's
            // offset mod ST, so a candidate is an ST-way select, not an
            // SPL-way one); the first (in (j, lane) order) whose resident's
            // other bucket is a split one (b < split or b > mask) is evicted --
            // under linear hashing those hold half the keys of the unsplit
            // buckets, so the chain likely ends there.  None: the rotating slot.
            constexpr int NC = VICTIM_LOOK / G > 0 ? (VICTIM_LOOK / G < SPL ? VICTIM_LOOK / G : SPL) : 1;
            constexpr int ST = SPL / NC;
            const int o = vrot % ST;
            uint64_t cand[NC];
            uint32_t good = 0, first_alt = 0;                // this lane's first good candidate's bucket
            bool found = false;
#pragma unroll
            for (int j = 0; j < NC; ++j) {
                uint64_t c = s[j * ST];
#pragma unroll
                for (int i = 1; i < ST; ++i)
                    if (i == o) c = s[j * ST + i];
                cand[j] = c;
                bool g = false;
                if (evicting && c != EMPTY) {
                    const uint32_t a = tv.alt(key_of(c), b);
                    g = a != b && (a < tv.split || a > tv.mask);
                    if (g && !found) {
                        first_alt = a;
                        found = true;
                    }
                }
                good |= wg.ballot(g) << (j * G);              // bit j * G + lane
            }
            int jv, lv;
            if (good) {
                const int f = __ffs(good) - 1;
                jv = f / G;
                lv = f % G;
            } else {                                         // the rotating slot (its offset is o)
                jv = (vrot % SPL) / ST;
                lv = vrot / SPL;
            }
            uint64_t w = cand[0];
#pragma unroll
            for (int j = 1; j < NC; ++j)
                if (j == jv) w = cand[j];
            vs = lv * SPL + jv * ST + o;
            victim = wg.bcast(w, lv);
            // the chosen (jv, lv) is lane lv's first good candidate (order is
            // j first), so its bucket is that lane's first_alt
            nb_alt = wg.bcast(first_alt, lv);
            alt_known = good != 0;
        } else {
            victim = wg.bcast(pick<SPL>(s, vs % SPL), vs / SPL);
        }
        const int vl = vs / SPL;
        const bool can = evicting && victim != EMPTY;
        // The victim's next bucket is known now: its load is issued right after
        // the swap CAS, so a round costs max(load, CAS) latency, not the sum.
        // A lost CAS discards the prefetched view (the round reloads b).
        const uint32_t nb = can ? (alt_known ? nb_alt : tv.alt(key_of(victim), b)) : b;
        uint64_t prev = victim;
        if (can && wg.gl == vl) {
            prev = cas64(tv.bucket(b) + vs, victim, kv);
            ab += 32;
        }
        const bool pf = can && r + 1 < max_evictions;       // the last round stashes instead
        if (pf) {
            load_slots<SPL>(wg.slot_ptr(tv.bucket(nb)), s);
            if (wg.gl == 0) ab += 256;
        }
        const bool ok = wg.bcast(can && wg.gl == vl && prev == victim, vl);
        if (evicting && ok) {
            const uint32_t hb = tv.addr(tv.h1(key_of(kv)));          // kv now lives in b
            if (wg.gl == 0 && hb != b) {
                atomicOr((unsigned long long*)&tv.spill[hb], (unsigned long long)spill_fp(key_of(kv)));
                ab += 8;
            }
            kv = victim;                                     // line 33
            b = nb;                                          // line 34: AltBucket
            have = pf;
            if (wg.gl == 0) ++evict;
        }
        if (busy) ++r;
        const bool finish = busy && (placed || r >= max_evictions);
        long long c1 = 0;
        if constexpr (PROF) c1 = clock64();
        if (finish && wg.gl == 0) {
            depth = r > depth ? r : depth;
            if (placed) ++st3;
            if (!placed) {                                   // Step 4: stash the in-hand entry
                const unsigned long long pos = atomicAdd(&sv.ctrl->stash_tail, 1ull);
                if (pos < sv.cap) {
                    atomicOr((unsigned long long*)&tv.spill[tv.addr(tv.h1(key_of(kv)))],
                             (unsigned long long)spill_fp(key_of(kv)));
                    sv.ring[pos] = kv;
                    stash_index_put(sv, key_of(kv), pos);
                    ++pushes;
                    ab += 8 + 8 + 8;
                } else {
                    ++lost;
                    if (status && !kvs) status[item] = 3;
                }
            }
        }
        if (finish) busy = false;
        if constexpr (PROF) {
            // the round is Step 3; the finish block is Step 4 when a group of
            // this warp pushed its in-hand entry to the stash
            const long long c2 = clock64();
            const bool pushed = __any_sync(FULL, finish && !placed);
            const unsigned long long s3 = warp_span(c0, c1), s4 = warp_span(c1, c2);
            if (lane == 0) {
                cyc3 += s3 + (pushed ? 0 : s4);
                cyc4 += pushed ? s4 : 0;
            }
        }
    }
    if constexpr (PROF) {
        block_add(&sv.ctrl->cyc[2], cyc3);
        block_add(&sv.ctrl->cyc[3], cyc4);
    }
    block_add(&sv.ctrl->evictions, evict);
    block_add(&sv.ctrl->stash_pushes, pushes);
    block_add(&sv.ctrl->failed, lost);
    block_add(&sv.ctrl->count, (unsigned long long)(0ull - lost));
    block_max(&sv.ctrl->max_depth, depth);
    block_add(&sv.ctrl->abytes[AB_EVICT], ab);
    block_add(&sv.ctrl->step3, st3);
}

template <int G, int MINB, bool PROF = false>
__global__ void __launch_bounds__(BLOCK, MINB)
k_insert_slow(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
              const uint64_t* __restrict__ kvs, const uint32_t* __restrict__ leftover,
              TableView tv, StashView sv, uint32_t max_evictions, uint8_t* __restrict__ status) {
    insert_slow_body<G, PROF>(keys, vals, kvs, leftover, tv, sv, max_evictions, status);
}

// --------------------------------------------------------------------------------
// Fused INSERT phase with owner election (cooperative, one launch).  The
// election of part q overlaps the insert fast path of part q-1: in every
// block, warps 6-7 elect (latency-bound L2 CASes) while warps 0-5 probe
// (HBM-bound), so the election's CAS round trips hide under the probes; a
// grid barrier separates the parts.  The two election tables alternate
// between parts and are never cleared inside the phase: a word is
//   epoch(6) | low 26 bits of fmix32(k ^ DEDUP_SEED) (its top 6 bits are the
//   part) | op(32),
// and a word whose epoch is not the current part's is empty.
// --------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t fused_owner(const uint64_t* tab, uint64_t mask, uint32_t hk26, uint32_t epoch,
                                                uint32_t self) {
    uint64_t h = hk26 & mask;
    for (uint64_t probe = 0; probe <= mask; ++probe) {
        const uint64_t e = tab[h];
        if ((uint32_t)(e >> 58) != epoch) return self;
        if (((uint32_t)(e >> 32) & 0x3FFFFFFu) == hk26) return (uint32_t)e;
        h = (h + 1) & mask;
    }
    return self;
}

template <int G>
__global__ void __launch_bounds__(BLOCK, 4)
k_insert_fused(const uint64_t* __restrict__ recs, const uint32_t* __restrict__ rvals,
               const uint64_t* __restrict__ part_info, uint64_t* __restrict__ tab0, uint64_t* __restrict__ tab1,
               uint64_t tab_mask, DedupView dd, TableView tv, StashView sv, uint8_t* __restrict__ status,
               uint32_t* __restrict__ vals_zero, uint32_t* __restrict__ leftover, uint32_t max_evictions,
               const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    constexpr int ELECT_WARPS = 2;                       // of WARPS_PER_BLOCK
    __shared__ uint32_t lbuf[WARPS_PER_BLOCK][32];
    WarpList wl{lbuf[threadIdx.x >> 5], 0};
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool elector = wib >= WARPS_PER_BLOCK - ELECT_WARPS;
    const uint64_t ew = (uint64_t)blockIdx.x * ELECT_WARPS + (wib - (WARPS_PER_BLOCK - ELECT_WARPS));
    const uint64_t n_ew = (uint64_t)gridDim.x * ELECT_WARPS;
    const uint64_t iw = (uint64_t)blockIdx.x * (WARPS_PER_BLOCK - ELECT_WARPS) + wib;
    const uint64_t n_iw = (uint64_t)gridDim.x * (WARPS_PER_BLOCK - ELECT_WARPS);
    const bool stash_on = sv.ctrl->stash_tail != 0;
    const uint32_t in_bytes = 8 + 4 + (status ? 1 : 0) + (vals_zero ? 4 : 0);
    FastState st;
    uint32_t eab = 0;
    unsigned long long eover = 0;
    for (uint32_t q = 0; q <= FUSED_PARTS; ++q) {
        if (elector && q < FUSED_PARTS) {                // ---- elect part q ----
            uint64_t* tab = (q & 1) ? tab1 : tab0;
            const uint64_t base = part_info[MAX_PARTS + q], cnt = part_info[q];
            for (uint64_t t0 = ew * 32; t0 < cnt; t0 += n_ew * 32) {
                const uint64_t t = t0 + lane;
                const bool active = t < cnt;
                const uint64_t rec = active ? recs[base + t] : EMPTY;
                const uint32_t k = (uint32_t)rec, op = (uint32_t)(rec >> 32);
                const uint32_t grp = __match_any_sync(FULL, k);
                if (!active) continue;
                eab += 8;
                uint32_t mx = op;
                if (__popc(grp) > 1) {                   // same key in this warp: pre-merge
                    dd.flag[op] = 1;
                    mx = __reduce_max_sync(grp, op);
                }
                if (op != mx) continue;
                const uint32_t hk26 = fmix32(k ^ DEDUP_SEED) & 0x3FFFFFFu;
                const uint64_t word = ((uint64_t)q << 58) | ((uint64_t)hk26 << 32) | op;
                uint64_t h = hk26 & tab_mask;
                uint64_t e = *(volatile uint64_t*)&tab[h];
                uint64_t probe = 0;
                while (true) {
                    if ((uint32_t)(e >> 58) != q) {          // stale epoch: free
                        const uint64_t prev = cas64(&tab[h], e, word);
                        eab += 32;
                        if (prev == e) break;
                        e = prev;                            // re-examine the same slot
                        continue;
                    }
                    if (((uint32_t)(e >> 32) & 0x3FFFFFFu) == hk26) {
                        dd.flag[op] = 1;
                        dd.flag[(uint32_t)e] = 1;
                        if (word > e) atomicMax((unsigned long long*)&tab[h], (unsigned long long)word);
                        eab += 32;
                        break;
                    }
                    if (++probe > tab_mask) { ++eover; break; }   // table full (never at the sizing)
                    h = (h + 1) & tab_mask;
                    e = *(volatile uint64_t*)&tab[h];
                }
            }
        }
        if (!elector && q >= 1) {                        // ---- insert part q-1 ----
            const uint32_t pq = q - 1;
            const uint64_t* tab = (pq & 1) ? tab1 : tab0;
            const uint64_t base = part_info[MAX_PARTS + pq], cnt = part_info[pq];
            auto fetch = [&](uint64_t tt, uint32_t& op, uint32_t& k, uint32_t& v) {
                const uint64_t rec = recs[tt];
                op = (uint32_t)(rec >> 32);
                k = (uint32_t)rec;
                v = rvals[tt];
            };
            auto owner = [&](const WarpGroup<G>& wg, bool valid, uint32_t k, uint32_t op, uint32_t& ab) {
                uint32_t own = op;
                if (valid && wg.gl == 0) {
                    ab += 1;
                    if (dd.flag[op]) {
                        own = fused_owner(tab, tab_mask, fmix32(k ^ DEDUP_SEED) & 0x3FFFFFFu, pq, op);
                        dd.owner_of[op] = own;
                        ab += 8 + 4;
                    }
                }
                return wg.bcast(own, 0) == op;
            };
            insert_fast_range<G, false>(base, base + cnt, iw, n_iw, fetch, owner, false, stash_on, in_bytes, tv, sv,
                                        status, vals_zero, leftover, wl, st);
        }
        grid.sync();
    }
    wl.flush(leftover, &sv.ctrl->n_left);
    block_add(&sv.ctrl->count, st.added);
    block_add(&sv.ctrl->abytes[AB_INSERT], st.ab);
    block_add(&sv.ctrl->abytes[AB_ELECT], eab);
    block_add(&sv.ctrl->eover, eover);
    grid.sync();
    // ---- Steps 3-4 for the leftovers ----
    insert_slow_body<G_SLOW, false>(keys, vals, nullptr, leftover, tv, sv, max_evictions, status);
    grid.sync();
    // ---- duplicates copy their owner's status (PHASED contract, A-17) ----
    const uint64_t total = part_info[MAX_PARTS + FUSED_PARTS - 1] + part_info[FUSED_PARTS - 1];
    for (uint64_t t = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; t < total; t += (uint64_t)gridDim.x * BLOCK) {
        const uint32_t op = (uint32_t)(recs[t] >> 32);
        if (!dd.flag[op]) continue;
        const uint32_t o = dd.owner_of[op];
        if (o != op && status) status[op] = status[o];
    }
}

int fused_grid(int num_sms) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)k_insert_fused<G_INSERT>, BLOCK, 0);
    return (nb > 0 ? nb : 1) * num_sms;
}

cudaError_t launch_insert_fused(int grid, cudaStream_t s, const uint64_t* recs, const uint32_t* rvals,
                                const uint64_t* part_info, uint64_t* tab0, uint64_t* tab1, uint64_t tab_mask,
                                DedupView dd, TableView tv, StashView sv, uint8_t* status, uint32_t* vals_zero,
                                uint32_t* leftover, uint32_t max_evictions, const uint32_t* keys,
                                const uint32_t* vals) {
    void* args[] = {(void*)&recs, (void*)&rvals, (void*)&part_info, (void*)&tab0, (void*)&tab1, (void*)&tab_mask,
                    (void*)&dd, (void*)&tv, (void*)&sv, (void*)&status, (void*)&vals_zero, (void*)&leftover,
                    (void*)&max_evictions, (void*)&keys, (void*)&vals};
    return cudaLaunchCooperativeKernel((const void*)k_insert_fused<G_INSERT>, grid, BLOCK, args, 0, s);
}

// --------------------------------------------------------------------------------
// ERASE (Alg. 4 ScanBucketAndDelete): WCME, winner CAS -> EMPTY;
// b2 only on a miss; then the stash.
// --------------------------------------------------------------------------------
template <int G, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB)
k_erase(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ idx, uint64_t n,
        const uint64_t* __restrict__ n_dev, TableView tv, StashView sv, DedupView dd,
        uint8_t* __restrict__ erased_out, uint32_t* __restrict__ vals_zero, DupFix fx) {
    using WG = WarpGroup<G>;
    constexpr int SPL = WG::SPL;
    WG wg;
    if (fx.flag) dup_fix(fx);               // the INSERT phase's duplicate fix-up (mixed batch)
    if (n_dev) n = *n_dev;
    const bool stash_on = sv.ctrl->stash_tail != 0;
    unsigned long long removed = 0;
    uint32_t ab = 0;                       // per-thread: < 2^32 bytes
    const uint64_t warp = ((uint64_t)blockIdx.x * BLOCK + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * BLOCK) >> 5;
    // software pipeline (as in k_find): the next iteration's (op, key) loads
    // are in flight while this one probes
    const uint64_t stride = nw * WG::GPW;
    uint32_t op_n = 0, k_n = INVALID_KEY;
    {
        const uint64_t t = warp * WG::GPW + wg.gi;
        if (t < n) {
            op_n = idx ? idx[t] : (uint32_t)t;
            k_n = keys[op_n];
        }
    }
    for (uint64_t t0 = warp * WG::GPW; t0 < n; t0 += stride) {
        const uint64_t t = t0 + wg.gi;
        const bool active = t < n;
        const uint32_t op = active ? op_n : 0u;                // < 2^32 (API)
        const uint32_t k = active ? k_n : INVALID_KEY;
        if (t + stride < n) {
            op_n = idx ? idx[t + stride] : (uint32_t)(t + stride);
            k_n = keys[op_n];
        }
        bool valid = k != INVALID_KEY;
        uint32_t b1 = 0, b2 = 0;
        if (valid) {
            b1 = tv.addr(tv.h1(k));
            b2 = tv.addr(tv.h2(k));
        }
        uint64_t s[SPL];
        uint64_t spill_w = 0;
        if (valid) {
            load_slots<SPL>(wg.slot_ptr(tv.bucket(b1)), s);
            spill_w = tv.spill[b1];
        } else {
            fill_empty<SPL>(s);
        }
        if (active && wg.gl == 0) {
            if (vals_zero) vals_zero[op] = 0;
            ab += 4 + (erased_out ? 1 : 0) + (vals_zero ? 4 : 0) + (idx ? 4 : 0) + (valid ? 256 + 8 : 0);
        }
        const bool owner = owns<G>(wg, dd, valid, k, op, ab);
        valid = valid && owner;
        bool done = wcme_cas<G>(wg, s, tv.bucket(b1), k, EMPTY, valid, ab);
        const bool maybe = valid && !done && (spill_w & spill_fp(k)) == spill_fp(k);
        const bool need2 = maybe && b2 != b1;
        if (__any_sync(FULL, need2)) {
            if (need2) load_slots<SPL>(wg.slot_ptr(tv.bucket(b2)), s);
            else fill_empty<SPL>(s);
            if (need2 && wg.gl == 0) ab += 256;
            done |= wcme_cas<G>(wg, s, tv.bucket(b2), k, EMPTY, need2, ab);
        }
        if (stash_on && maybe && !done && wg.gl == 0) {
            uint64_t sw;
            ab += 16;
            int64_t pos = stash_lookup(sv, k, &sw);
            while (pos >= 0) {
                uint64_t prev = cas64(&sv.ring[pos], sw, EMPTY);
                if (prev == sw) { done = true; break; }
                pos = stash_lookup(sv, k, &sw);
            }
        }
        if (active && wg.gl == 0 && owner) {
            if (erased_out) erased_out[op] = done ? 1 : 0;
            if (done) ++removed;
        }
    }
    block_add(&sv.ctrl->count, 0ull - removed);
    block_add(&sv.ctrl->abytes[AB_ERASE], ab);
}

// --------------------------------------------------------------------------------
// NEXT-4: the monolithic concurrent mixed kernel (the paper's
// single-kernel model).  One cooperative launch per mixed
// batch; its stages are separated by grid-wide barriers:
//   0. clear the per-batch group table and duplicate flags;
//   1. per-key group election: all inserts of a key form one insert group and
//      all erases one erase group; the highest op index of a group is its
//      owner (A-15: without it, same-key inserts would both claim a slot);
//   2. every op runs CONCURRENTLY in one pass, finds, erases and inserts
//      interleaved in the same warps: finds read b1 (b2 / stash only when the
//      spill word allows), group owners apply their group as ONE atomic
//      operation (erase: CAS -> EMPTY; insert: replace CAS or a blocking
//      claim CAS with the owner's value), inserts whose candidate buckets are
//      both full go to the leftover list;
//   3. bounded eviction + stash for the leftovers (Steps 3-4), i.e. AFTER
//      every find and erase of the batch: no lookup can observe an entry in
//      an eviction chain's hand (A-16), so no seqlock is needed;
//   4. duplicates copy their group owner's result.
// Contract (include/hive.h hive_mixed_concurrent): every op of a key takes
// effect atomically in some order -- the batch is linearizable per key with
// each group one atomic step whose members all report the presence before
// the group.  Single-type batches therefore give exactly the PHASED results.
// --------------------------------------------------------------------------------
constexpr uint32_t MONO_ERASE_BIT = 0x80000000u;   // group class in the table word's op field
__device__ __forceinline__ uint32_t mono_hash(uint32_t k, uint32_t cls) {
    return fmix32(k ^ DEDUP_SEED ^ (cls ? 0x9E3779B9u : 0u));
}
// Owner (highest op) of the (k, cls) group; `self` if the table has no entry.
__device__ __forceinline__ uint32_t mono_owner(const uint64_t* tab, uint64_t mask, uint32_t k, uint32_t cls,
                                               uint32_t self) {
    uint64_t h = mono_hash(k, cls) & mask;
    const uint32_t tag = cls ? MONO_ERASE_BIT : 0u;
    for (uint64_t probe = 0; probe <= mask; ++probe) {
        const uint64_t e = tab[h];
        if (e == EMPTY) return self;
        if ((uint32_t)(e >> 32) == k && ((uint32_t)e & MONO_ERASE_BIT) == tag) return (uint32_t)e & ~MONO_ERASE_BIT;
        h = (h + 1) & mask;
    }
    return self;
}

template <int G, int GS>
__global__ void __launch_bounds__(BLOCK, 4)
k_mixed_mono(const uint8_t* __restrict__ opc, const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
             uint64_t n, TableView tv, StashView sv, uint64_t* __restrict__ tab, uint64_t tab_mask,
             uint8_t* __restrict__ flag, uint32_t* __restrict__ owner_of, uint32_t* __restrict__ leftover,
             uint32_t max_evictions, uint8_t* __restrict__ result, uint32_t* __restrict__ vals_out) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const uint64_t tid = (uint64_t)blockIdx.x * BLOCK + threadIdx.x;
    const uint64_t nthreads = (uint64_t)gridDim.x * BLOCK;
    const int lane = threadIdx.x & 31;
    // ---- stage 0: clear ----
    for (uint64_t i = tid; i <= tab_mask; i += nthreads) tab[i] = EMPTY;
    for (uint64_t i = tid; i < n; i += nthreads) flag[i] = 0;
    grid.sync();
    // ---- stage 1: group election (insert-if-absent, atomicMax keeps the max op) ----
    uint32_t ab = 0;
    for (uint64_t t0 = tid & ~31ull; t0 < n; t0 += nthreads) {
        const uint64_t t = t0 + lane;
        const uint32_t o = t < n ? opc[t] : 0u;
        const uint32_t k = t < n ? keys[t] : INVALID_KEY;
        const bool part = t < n && (o == 1 || o == 2) && k != INVALID_KEY;
        const uint32_t cls = o == 2 ? 1u : 0u;
        // lanes of this warp with the same (key, class): pre-reduce to the max op
        const uint32_t grp = __match_any_sync(FULL, part ? ((uint64_t)k << 1 | cls) : ~0ull);
        if (!part) continue;
        if (__popc(grp) > 1) flag[t] = 1;
        if ((31 - __clz(grp)) != lane) continue;
        const uint64_t word = ((uint64_t)k << 32) | (cls ? MONO_ERASE_BIT : 0u) | (uint32_t)t;
        uint64_t h = mono_hash(k, cls) & tab_mask;
        for (uint64_t probe = 0; probe <= tab_mask; ++probe) {
            const uint64_t prev = cas64(&tab[h], EMPTY, word);
            ab += 32;
            if (prev == EMPTY) break;
            if ((prev >> 32) == k && (((uint32_t)prev & MONO_ERASE_BIT) != 0) == (cls != 0)) {
                flag[t] = 1;
                flag[(uint32_t)prev & ~MONO_ERASE_BIT] = 1;
                if (word > prev) atomicMax((unsigned long long*)&tab[h], (unsigned long long)word);
                break;
            }
            h = (h + 1) & tab_mask;
        }
    }
    grid.sync();
    // ---- stage 2: all ops concurrently (one G-lane group per op) ----
    {
        using WG = WarpGroup<G>;
        constexpr int SPL = WG::SPL;
        __shared__ uint32_t lbuf[WARPS_PER_BLOCK][32];
        WG wg;
        WarpList wl{lbuf[threadIdx.x >> 5], 0};
        const bool stash_on = sv.ctrl->stash_tail != 0;
        unsigned long long added = 0, removed = 0;
        const uint64_t warp = tid >> 5, nw = nthreads >> 5;
        const uint64_t stride = nw * WG::GPW;
        bool pend = false;                       // optimistic claim issued last iteration
        uint64_t pend_prev = EMPTY;
        uint32_t pend_item = 0;
        // software pipeline: the next iteration's (opcode, key, value) loads are
        // in flight while this iteration probes
        uint32_t o_n = 3u, k_n = INVALID_KEY, v_n = 0;
        auto fetch = [&](uint64_t tt) {
            o_n = tt < n ? opc[tt] : 3u;
            k_n = tt < n ? keys[tt] : INVALID_KEY;
            v_n = tt < n ? vals[tt] : 0u;
        };
        fetch(warp * WG::GPW + wg.gi);
        for (uint64_t base = warp * WG::GPW; base < n; base += stride) {
            const uint64_t t = base + wg.gi;
            const bool active = t < n;
            const uint32_t o = active ? o_n : 3u;
            const uint32_t k = active ? k_n : INVALID_KEY;
            const uint32_t v = o == 1 ? v_n : 0u;
            fetch(t + stride);
            bool valid = o < 3 && k != INVALID_KEY;
            if (active && wg.gl == 0) {
                vals_out[t] = 0;
                if (!valid) result[t] = (o == 1) ? 2 : 0;        // reserved key / unknown opcode
                ab += 4 + 1 + 1 + 4 + (o == 1 ? 4 : 0);
            }
            // group members other than the owner only copy its result (stage 4)
            uint32_t own = (uint32_t)t;
            if (valid && o != 0 && wg.gl == 0 && flag[t]) {
                own = mono_owner(tab, tab_mask, k, o == 2 ? 1u : 0u, (uint32_t)t);
                owner_of[t] = own;
            }
            if (wg.bcast(own, 0) != (uint32_t)t) valid = false;
            const bool is_find = valid && o == 0, is_ins = valid && o == 1, is_era = valid && o == 2;
            uint32_t b1 = 0, b2 = 0, h2 = 0;
            if (valid) {
                b1 = tv.addr(tv.h1(k));
                h2 = tv.h2(k);
                b2 = tv.addr(h2);
            }
            const uint32_t lrot = c_claim_rot >= 1 ? (h2 >> 24) % G : 0u;
            const uint32_t srot = c_claim_rot >= 2 ? (h2 >> 27) % SPL : 0u;
            const uint64_t fp = spill_fp(k), kv = pack(k, v);
            // one bucket view (b1, later possibly b2), as in k_insert_fast
            uint64_t sl[SPL];
            uint64_t spill_w = 0;
            int jm1 = SPL, jf1 = SPL;
            if (valid) {
                load_slots<SPL>(wg.slot_ptr(tv.bucket(b1)), sl);
                spill_w = tv.spill[b1];
                if (wg.gl == 0) ab += 256 + 8;
                scan_slots_rot<SPL>(sl, k, srot, jm1, jf1);
            } else {
                fill_empty<SPL>(sl);
            }
            // WCME on b1: finds read, erase / insert owners CAS the match
            uint32_t val = 0;
            bool done = wcme_value<G>(wg, sl, k, is_find, &val);
            if (__any_sync(FULL, (is_ins || is_era) && jm1 < SPL))
                done |= wcme_cas<G>(wg, sl, tv.bucket(b1), k, is_era ? EMPTY : kv, is_ins || is_era, ab);
            const bool maybe = valid && !done && (spill_w & fp) == fp;
            const bool need2 = maybe && b2 != b1;
            bool have2 = false;
            if (__any_sync(FULL, need2)) {
                if (need2) load_slots<SPL>(wg.slot_ptr(tv.bucket(b2)), sl);
                else fill_empty<SPL>(sl);
                if (need2 && wg.gl == 0) ab += 256;
                have2 = need2;
                done |= wcme_value<G>(wg, sl, k, need2 && is_find, &val);
                done |= wcme_cas<G>(wg, sl, tv.bucket(b2), k, is_era ? EMPTY : kv, need2 && !is_find, ab);
            }
            if (stash_on) {
                bool sdone = false;
                uint32_t sval = 0;
                if (maybe && !done && wg.gl == 0) {
                    uint64_t sw;
                    ab += 16;
                    int64_t pos = stash_lookup(sv, k, &sw);
                    if (is_find) {
                        if (pos >= 0) { sdone = true; sval = val_of(sw); }
                    } else {
                        while (pos >= 0) {
                            const uint64_t prev = cas64(&sv.ring[pos], sw, is_era ? EMPTY : kv);
                            if (prev == sw) { sdone = true; break; }
                            pos = stash_lookup(sv, k, &sw);
                        }
                    }
                }
                sdone = wg.bcast(sdone, 0);
                sval = wg.bcast(sval, 0);
                if (sdone && is_find) val = sval;
                done |= sdone;
            }
            // resolve last iteration's optimistic claim: a lost one goes to
            // the Step 3-4 stage (an insert placed there is linearized after
            // every find and erase of the batch, when its key is still absent)
            wl.push(pend && pend_prev != EMPTY, pend_item, leftover, &sv.ctrl->n_left);
            pend = false;
            // inserts of absent keys: optimistic WABC claim in b1 at the slot the
            // Step-1 scan found free, then b2 (first-fit, A-21), as k_insert_fast
            const bool want1 = is_ins && !done;
            bool placed = wabc_claim_issue<G>(wg, jf1, tv.bucket(b1), kv, want1, pend, pend_prev, pend_item,
                                              (uint32_t)t, ab, lrot);
            const bool want2 = want1 && !placed && b2 != b1;
            if (__any_sync(FULL, want2)) {
                if (want2 && !have2) load_slots<SPL>(wg.slot_ptr(tv.bucket(b2)), sl);
                if (want2 && !have2 && wg.gl == 0) ab += 256;
                int jm2, jf2 = SPL;
                if (want2) scan_slots<SPL>(sl, INVALID_KEY, jm2, jf2);
                const bool p2 = wabc_claim_issue<G>(wg, jf2, tv.bucket(b2), kv, want2, pend, pend_prev, pend_item,
                                                    (uint32_t)t, ab, lrot);
                if (p2 && wg.gl == 0) {
                    atomicOr((unsigned long long*)&tv.spill[b1], (unsigned long long)fp);
                    ab += 8;
                }
                placed |= p2;
            }
            if (valid && wg.gl == 0) {
                if (is_find) {
                    result[t] = done ? 1 : 0;
                    vals_out[t] = done ? val : 0u;
                } else {
                    result[t] = done ? 1 : 0;                 // presence before the group
                    if (is_ins && !done) ++added;
                    if (is_era && done) ++removed;
                }
            }
            wl.push(want1 && !placed && wg.gl == 0, (uint32_t)t, leftover, &sv.ctrl->n_left);
        }
        wl.push(pend && pend_prev != EMPTY, pend_item, leftover, &sv.ctrl->n_left);
        wl.flush(leftover, &sv.ctrl->n_left);
        block_add(&sv.ctrl->count, added - removed);
    }
    block_add(&sv.ctrl->abytes[AB_INSERT], ab);
    grid.sync();
    // ---- stage 3: Steps 3-4 for the leftovers, after every find and erase ----
    insert_slow_body<GS, false>(keys, vals, nullptr, leftover, tv, sv, max_evictions, result);
    grid.sync();
    // ---- stage 4: group members copy their owner's result ----
    for (uint64_t t = tid; t < n; t += nthreads)
        if (flag[t] && opc[t] != 0 && keys[t] != INVALID_KEY) {
            const uint32_t own = owner_of[t];
            if (own != (uint32_t)t) result[t] = result[own];
        }
}

// Duplicates copy their owner's outcome (PHASED contract, A-17): the dense
// form scans flag[0, n) (16 flags per load); flags are set only for the
// phase's own ops.  Also run as the prologue of the next phase's kernel in a
// mixed batch (DupFix): the two touch result entries of different op classes.
__global__ void __launch_bounds__(BLOCK)
k_dup_copy(const uint32_t* __restrict__ idx, uint64_t n, const uint64_t* __restrict__ n_dev,
           DedupView dd, uint8_t* __restrict__ out) {
    if (dd.any && *dd.any == 0) return;     // the election flagged nothing
    if (n_dev) n = *n_dev;
    if (!idx) {
        dup_fix(DupFix{dd.flag, dd.owner_of, dd.any, out, n});
        return;
    }
    for (uint64_t t = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * BLOCK) {
        const uint64_t op = idx[t];
        if (!dd.flag[op]) continue;
        const uint32_t o = dd.owner_of[op];
        if (o != (uint32_t)op) out[op] = out[o];
    }
}

// --------------------------------------------------------------------------------
// Linear-hashing split: one warp per (b_src, b_dst) pair, one
// lane per slot as in the paper's listing.  The destination bucket is written
// whole (movers compacted into slots 0..n-1, EMPTY after), so new buckets need
// no separate initialisation.  Residence hash: reading A-3.
// --------------------------------------------------------------------------------
__global__ void __launch_bounds__(BLOCK)
k_split(TableView tv, uint32_t n_pairs, Ctrl* ctrl) {
    const uint32_t pair = (blockIdx.x * BLOCK + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (pair >= n_pairs) return;
    const uint32_t b_src = tv.split + pair;
    const uint32_t b_dst = b_src + tv.mask + 1u;
    const uint32_t next_mask = (tv.mask << 1) | 1u;
    uint64_t* src = tv.bucket(b_src);
    uint64_t* dst = tv.bucket(b_dst);
    const uint64_t kv = src[lane];
    bool should_move = false;
    if (kv != EMPTY) {
        const uint32_t k = key_of(kv);
        const uint32_t h1 = tv.h1(k);
        const uint32_t h = ((h1 & tv.mask) == b_src) ? h1 : tv.h2(k);
        should_move = (h & next_mask) == b_dst;
    }
    const uint32_t move_mask = __ballot_sync(FULL, should_move);
    const uint32_t my_rank = __popc(move_mask & lanemask_lt());
    const int n_movers = __popc(move_mask);
    if (should_move) {
        dst[my_rank] = kv;
        src[lane] = EMPTY;
    }
    if (lane >= n_movers) dst[lane] = EMPTY;                      // rest of the new bucket
    // keys whose b1 was b_src may now have b1 = b_dst: the new bucket inherits
    // the spill word (conservative)
    if (lane == 0) tv.spill[b_dst] = tv.spill[b_src];
}

// Contraction, LIFO pairs t = 0..n_pairs-1 with
// b_dst = split-1-t, b_src = b_dst + 2^m.  Pass 1 finds the first pair that
// must abort (n_move > n_free) -> *abort_at (initialised to n_pairs
// by the host); pass 2 merges the pairs before it (the sequential LIFO loop
// stops at its first abort, reading A-25).  A segment whose predecessor
// segment (the previous linear-hashing round of the same shrink phase)
// aborted merges nothing.
__global__ void __launch_bounds__(BLOCK)
k_merge_check(TableView tv, uint32_t n_pairs, unsigned long long* abort_at,
              const unsigned long long* prev_abort, uint64_t prev_pairs) {
    const uint32_t t = (blockIdx.x * BLOCK + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= n_pairs) return;
    if (prev_abort && *prev_abort < prev_pairs) {
        if (t == 0 && lane == 0) *abort_at = 0;
        return;
    }
    const uint32_t b_dst = tv.split - 1u - t;
    const uint32_t b_src = b_dst + tv.mask + 1u;
    const uint32_t occ = __ballot_sync(FULL, tv.bucket(b_src)[lane] != EMPTY);
    const uint32_t fre = __ballot_sync(FULL, tv.bucket(b_dst)[lane] == EMPTY);
    if (lane == 0 && __popc(occ) > __popc(fre)) atomicMin(abort_at, (unsigned long long)t);
}
__global__ void __launch_bounds__(BLOCK)
k_merge_apply(TableView tv, uint32_t n_pairs, const unsigned long long* abort_at) {
    const uint32_t t = (blockIdx.x * BLOCK + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= n_pairs || t >= *abort_at) return;
    const uint32_t b_dst = tv.split - 1u - t;
    const uint32_t b_src = b_dst + tv.mask + 1u;
    uint64_t* src = tv.bucket(b_src);
    uint64_t* dst = tv.bucket(b_dst);
    const uint64_t kv = src[lane];
    const bool live = kv != EMPTY;
    const uint32_t occ_mask = __ballot_sync(FULL, live);
    const uint32_t my_rank = __popc(occ_mask & lanemask_lt());
    const uint32_t dst_free = __ballot_sync(FULL, dst[lane] == EMPTY);
    if (live) {
        // pos = select_nth_one(dst_free, my_rank)
        uint32_t m = dst_free;
        for (uint32_t r = 0; r < my_rank; ++r) m &= m - 1;
        const int pos = __ffs(m) - 1;
        dst[pos] = kv;
        src[lane] = EMPTY;
    }
    if (lane == 0) tv.spill[b_dst] |= tv.spill[b_src];           // spill words merge
}

// --------------------------------------------------------------------------------
// misc: dump, stats, partition / routing
// --------------------------------------------------------------------------------
__global__ void __launch_bounds__(BLOCK)
k_dump(TableView tv, uint64_t n_slots, StashView sv, uint64_t ring_n, uint32_t* __restrict__ keys,
       uint32_t* __restrict__ vals, uint64_t cap) {
    const uint64_t total = n_slots + ring_n;
    const uint64_t stride = (uint64_t)gridDim.x * BLOCK;
    for (uint64_t i0 = (uint64_t)blockIdx.x * BLOCK + (threadIdx.x & ~31u); i0 < total; i0 += stride) {
        const uint64_t i = i0 + (threadIdx.x & 31);
        uint64_t w = EMPTY;
        if (i < n_slots) w = tv.buckets[i];
        else if (i < total) w = sv.ring[i - n_slots];
        const bool live = w != EMPTY;
        const uint32_t bal = __ballot_sync(FULL, live);
        unsigned long long base = 0;
        if ((threadIdx.x & 31) == 0 && bal) base = atomicAdd(&sv.ctrl->dump_n, (unsigned long long)__popc(bal));
        base = __shfl_sync(FULL, base, 0);
        if (live) {
            const uint64_t p = base + __popc(bal & lanemask_lt());
            if (p < cap) {
                keys[p] = key_of(w);
                vals[p] = val_of(w);
            }
        }
    }
}

__global__ void __launch_bounds__(BLOCK)
k_count_b1(TableView tv, uint64_t n_slots, Ctrl* ctrl) {
    unsigned long long c = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; i < n_slots;
         i += (uint64_t)gridDim.x * BLOCK) {
        const uint64_t w = tv.buckets[i];
        if (w != EMPTY && tv.addr(tv.h1(key_of(w))) == (uint32_t)(i / SLOTS)) ++c;
    }
    block_add(&ctrl->in_b1, c);
}

// shard(k) = (fmix32(k ^ seed) * G) >> 32 of op i
__device__ __forceinline__ uint32_t shard_of(uint32_t n_parts, uint32_t seed, const uint32_t* keys, uint64_t i) {
    return (uint32_t)(((uint64_t)fmix32(keys[i] ^ seed) * (uint64_t)n_parts) >> 32);
}

// Lanes of the warp holding the same label q (all lanes call).  Labels below
// 16 (routing: <= 8 shards + the out-of-range label) take 4
// ballots; larger label sets use __match_any_sync (measured ~3x slower).
__device__ __forceinline__ uint32_t same_label(uint32_t q, bool small) {
    if (!small) return __match_any_sync(FULL, q);
    uint32_t g = FULL;
#pragma unroll
    for (int bit = 0; bit < 4; ++bit) {
        const uint32_t b = __ballot_sync(FULL, (q >> bit) & 1u);
        g &= ((q >> bit) & 1u) ? b : ~b;
    }
    return g;
}

// Stable partition pass 1: per-warp, per-part counts (part-major layout).
__global__ void __launch_bounds__(BLOCK)
k_part_count(int mode, uint32_t n_parts, uint32_t seed, const uint32_t* __restrict__ keys,
             const uint8_t* __restrict__ ops, uint64_t n, uint64_t n_warps,
             uint64_t* __restrict__ cnt, const uint32_t* __restrict__ idx,
             const uint64_t* __restrict__ n_dev, uint32_t chunk) {
    if (n_dev) n = *n_dev;
    __shared__ uint32_t sc[WARPS_PER_BLOCK][MAX_PARTS + 1];
    const bool small = n_parts < 16;
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t w = (uint64_t)blockIdx.x * WARPS_PER_BLOCK + wib;
    for (int p = lane; p <= MAX_PARTS; p += 32) sc[wib][p] = 0;
    __syncwarp();
    if (w < n_warps) {
        const uint64_t lo = w * chunk;
        const uint64_t hi = lo + chunk < n ? lo + chunk : (lo < n ? n : lo);
        // PART_UNROLL rows of 32 elements per iteration: their loads are all
        // issued before the first label is ranked
        for (uint64_t i0 = lo; i0 < hi; i0 += 32 * PART_UNROLL) {
            uint32_t pp[PART_UNROLL];
#pragma unroll
            for (int u = 0; u < PART_UNROLL; ++u) {
                const uint64_t i = i0 + u * 32 + lane;
                const uint64_t e = i < hi ? (idx ? (uint64_t)idx[i] : i) : 0;
                pp[u] = i < hi ? shard_of(n_parts, seed, keys, e) : MAX_PARTS;
            }
#pragma unroll
            for (int u = 0; u < PART_UNROLL; ++u) {
                uint32_t p = pp[u];
                if (small && p >= n_parts) p = MAX_PARTS;
                const uint32_t grp = same_label(small && p == MAX_PARTS ? 15u : p, small);
                if ((__ffs(grp) - 1) == lane) sc[wib][p] += __popc(grp);
                __syncwarp();
            }
        }
        for (uint32_t p = lane; p < n_parts; p += 32) cnt[(uint64_t)p * n_warps + w] = sc[wib][p];
    }
}

// Pass 2: exclusive scan over cnt (single block).  Tiles of 1024 threads x
// SCAN_ITEMS consecutive elements: each thread scans its items serially, the
// thread totals are scanned with warp shuffles, the warp totals by warp 0.
// part_info[p] = total of part p, part_info[MAX_PARTS + p] = start of part p.
constexpr int SCAN_ITEMS = 8;
__global__ void __launch_bounds__(1024)
k_part_scan(uint64_t* __restrict__ cnt, uint64_t E, uint32_t n_parts, uint64_t n_warps,
            uint64_t* __restrict__ part_info) {
    __shared__ uint64_t wsum[32];
    __shared__ uint64_t carry;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    constexpr uint64_t TILE = 1024ull * SCAN_ITEMS;
    for (uint64_t base = 0; base < E; base += TILE) {
        const uint64_t i0 = base + (uint64_t)tid * SCAN_ITEMS;
        uint64_t v[SCAN_ITEMS];
        uint64_t t = 0;
#pragma unroll
        for (int j = 0; j < SCAN_ITEMS; ++j) {
            v[j] = i0 + j < E ? cnt[i0 + j] : 0;
            t += v[j];
        }
        uint64_t x = t;                                   // inclusive warp scan of thread totals
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint64_t w = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t y = __shfl_up_sync(FULL, w, o);
                if (lane >= o) w += y;
            }
            wsum[lane] = w;
        }
        __syncthreads();
        uint64_t run = carry + (wid ? wsum[wid - 1] : 0) + x - t;
#pragma unroll
        for (int j = 0; j < SCAN_ITEMS; ++j) {
            if (i0 + j < E) cnt[i0 + j] = run;
            run += v[j];
        }
        __syncthreads();
        if (tid == 0) carry += wsum[31];
        __syncthreads();
    }
    const uint64_t total = carry;
    if (tid < (int)n_parts) {
        const uint64_t start = n_warps ? cnt[(uint64_t)tid * n_warps] : 0;
        const uint64_t end = (tid + 1 < (int)n_parts) ? cnt[(uint64_t)(tid + 1) * n_warps] : total;
        part_info[tid] = end - start;
        part_info[MAX_PARTS + tid] = start;
    }
}

// Pass 3: stable scatter.  CLASSIFY writes op indices into per-part regions
// out_idx + p * idx_stride (invalid opcodes: result 0 / value 0 in place).
// ROUTE writes packed records, opcodes and the inverse positions.
__global__ void __launch_bounds__(BLOCK)
k_part_scatter(int mode, uint32_t n_parts, uint32_t seed, const uint32_t* __restrict__ keys,
               const uint32_t* __restrict__ vals, const uint8_t* __restrict__ ops, uint64_t n,
               uint64_t n_warps, const uint64_t* __restrict__ off,
               const uint64_t* __restrict__ part_info, uint64_t* __restrict__ send_kv,
               uint8_t* __restrict__ send_ops, uint32_t* __restrict__ pos_out, const uint32_t* __restrict__ idx,
               const uint64_t* __restrict__ n_dev, uint32_t chunk, PeerDest pd) {
    __shared__ uint64_t run[WARPS_PER_BLOCK][MAX_PARTS + 1];
    const bool small = n_parts < 16;
    if (n_dev) n = *n_dev;
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t w = (uint64_t)blockIdx.x * WARPS_PER_BLOCK + wib;
    if (w >= n_warps) return;
    for (uint32_t p = lane; p < n_parts; p += 32) run[wib][p] = off[(uint64_t)p * n_warps + w];
    __syncwarp();
    const uint64_t lo = w * chunk;
    const uint64_t hi = lo + chunk < n ? lo + chunk : (lo < n ? n : lo);
    for (uint64_t r0 = lo; r0 < hi; r0 += 32 * PART_UNROLL) {
        uint32_t pp[PART_UNROLL];
        uint64_t ee[PART_UNROLL];
#pragma unroll
        for (int u = 0; u < PART_UNROLL; ++u) {                  // all rows' loads first
            const uint64_t i = r0 + u * 32 + lane;
            ee[u] = i < hi ? (idx ? (uint64_t)idx[i] : i) : 0;
            pp[u] = i < hi ? shard_of(n_parts, seed, keys, ee[u]) : MAX_PARTS;
        }
#pragma unroll
        for (int u = 0; u < PART_UNROLL; ++u) {                  // then rank the rows in order
            const uint64_t i0 = r0 + u * 32;
            const uint64_t i = i0 + lane;
            const bool in = i < hi;
            const uint64_t e = ee[u];
            uint32_t p = pp[u];
            if (small && p >= n_parts) p = MAX_PARTS;
            const uint32_t grp = same_label(small && p == MAX_PARTS ? 15u : p, small);
            const uint32_t rank = __popc(grp & lanemask_lt());
            uint64_t pos = 0;
            if (in && p < n_parts) pos = run[wib][p] + rank;
            __syncwarp();
            if (in && p < n_parts && (__ffs(grp) - 1) == lane) run[wib][p] += __popc(grp);
            __syncwarp();
            if (!in) continue;
            if (mode == PART_ROUTE_KEYS) {
                reinterpret_cast<uint32_t*>(send_kv)[pos] = keys[i];
                pos_out[i] = (uint32_t)pos;
            } else if (mode == PART_ROUTE_PAD) {
                // region p of the padded NCCL send buffer (pd.region = cap
                // records); an op past the region's capacity is not sent
                // (over an index list -- source-side election -- op e is the
                // list entry i; pos_out is indexed by the list position)
                const uint64_t rel = pos - part_info[MAX_PARTS + p];
                if (rel < pd.region) {
                    const uint64_t at = (uint64_t)p * pd.region + rel;
                    send_kv[at] = ((uint64_t)(vals ? vals[e] : 0u) << 32) | keys[e];
                    if (send_ops) send_ops[at] = ops[e];
                    pos_out[i] = (uint32_t)at;
                } else {
                    pos_out[i] = NO_POS;
                }
            } else if (mode == PART_ROUTE_P2P) {
                // owner p's inbox, this rank's region: a remote store over NVLink
                // (a local one when p is this rank); the stable rank keeps the
                // (rank, index) order the owner's PHASED batch relies on
                // (an op past the region's capacity is not sent: pos = NO_POS)
                const uint64_t rel = pos - part_info[MAX_PARTS + p];
                if (rel < pd.region) {
                    const uint64_t at = (uint64_t)pd.rank * pd.region + rel;
                    pd.kv[p][at] = ((uint64_t)(vals ? vals[i] : 0u) << 32) | keys[i];
                    if (pd.ops[p]) pd.ops[p][at] = ops[i];
                    pos_out[i] = (uint32_t)((uint64_t)p * pd.region + rel);
                } else {
                    pos_out[i] = NO_POS;
                }
            } else {
                send_kv[pos] = ((uint64_t)(vals ? vals[i] : 0u) << 32) | keys[i];
                if (send_ops) send_ops[pos] = ops[i];
                pos_out[i] = (uint32_t)pos;
            }
        }
    }
    // peer stores are made visible system-wide before the phase signal
    // (k_p2p_signal runs after this kernel in stream order)
    if (mode == PART_ROUTE_P2P) __threadfence_system();
}

__global__ void __launch_bounds__(BLOCK)
k_unroute(const uint32_t* __restrict__ pos, uint64_t n, const uint8_t* __restrict__ in8,
          uint8_t* __restrict__ out8, const uint32_t* __restrict__ in32, uint32_t* __restrict__ out32) {
    for (uint64_t i = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (uint64_t)gridDim.x * BLOCK) {
        const uint32_t p = pos[i];
        if (out8) out8[i] = in8[p];
        if (out32) out32[i] = in32[p];
    }
}

__global__ void __launch_bounds__(BLOCK)
k_unpack(const uint64_t* __restrict__ kv, uint64_t n, uint32_t* __restrict__ keys,
         uint32_t* __restrict__ vals) {
    for (uint64_t i = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (uint64_t)gridDim.x * BLOCK) {
        const uint64_t w = kv[i];
        if (keys) keys[i] = key_of(w);
        if (vals) vals[i] = val_of(w);
    }
}

// Calibration ceiling (SURVEY §8(d) "Calibration ceiling"): the pure gather a
// probe reduces to.  Per op: read a 4 B key, pick a 256 B block by the
// multiply-high reduction of fmix32(key), load it with the same group loads as
// k_find (G lanes, 256-bit vectors), write one 4 B word (xor of the block).  No
// compares, no second probe: random 256 B reads at the find kernel's access
// count, against which the probe kernels' GB/s is judged.
// mode 1 adds a plain 8 B store and mode 2 a 64-bit CAS (with return) into
// one slot of each gathered block: the read/write mix of an insert probe.
template <int G, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB)
k_gather(const uint32_t* __restrict__ keys, uint64_t n, const uint64_t* __restrict__ blocks,
         uint64_t n_blocks, uint32_t* __restrict__ out, uint32_t mode) {
    using WG = WarpGroup<G>;
    constexpr int SPL = WG::SPL;
    WG wg;
    const uint64_t warp = ((uint64_t)blockIdx.x * BLOCK + threadIdx.x) >> 5;
    const uint64_t stride = (((uint64_t)gridDim.x * BLOCK) >> 5) * WG::GPW;
    uint64_t t = warp * WG::GPW + wg.gi;
    uint32_t k_n = t < n ? keys[t] : 0u;
    for (uint64_t t0 = warp * WG::GPW; t0 < n; t0 += stride) {
        t = t0 + wg.gi;
        const uint32_t k = k_n;
        if (t + stride < n) k_n = keys[t + stride];
        uint64_t s[SPL];
        uint32_t x = 0;
        if (t < n) {
            const uint64_t b = ((uint64_t)fmix32(k) * n_blocks) >> 32;
            uint64_t* blk = const_cast<uint64_t*>(blocks) + b * SLOTS;
            if (mode) load_slots<SPL>(blk + wg.gl * SPL, s);
            else load_slots_ro<SPL>(blk + wg.gl * SPL, s);
#pragma unroll
            for (int j = 0; j < SPL; ++j) x ^= (uint32_t)s[j] ^ (uint32_t)(s[j] >> 32);
            if (mode && wg.gl == 0) {
                const int j = (int)(k & 31u);              // one slot, one dirty sector
                if (mode == 1) blk[j] = s[0] ^ 1ull;
                else x ^= (uint32_t)cas64(blk + j, s[0], s[0] ^ 1ull);
            }
        }
#pragma unroll
        for (int o = 1; o < G; o <<= 1) x ^= __shfl_xor_sync(FULL, x, o);
        if (t < n && wg.gl == 0) out[t] = x;
    }
}

// --------------------------------------------------------------------------------
// launchers
// --------------------------------------------------------------------------------
static int occ(const void* fn) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, BLOCK, 0);
    return nb > 0 ? nb : 1;
}

static int env_g(const char* name, int dflt) {
    const char* e = getenv(name);
    if (!e) return dflt;
    const int g = atoi(e);
    return (g == 2 || g == 4 || g == 8) ? g : dflt;
}

#define HIVE_DISPATCH_G(g, X) \
    switch (g) {              \
        case 1: X(1); break;  \
        case 2: X(2); break;  \
        case 4: X(4); break;  \
        default: X(8); break; \
    }

#define HIVE_SWITCH_G(g, mb, X) \
    switch (g) {                  \
        case 2: X(2, mb); break;  \
        case 4: X(4, mb); break;  \
        default: X(8, mb); break; \
    }
#define HIVE_DISPATCH_GM(g, mb, X)                     \
    if (mb >= 6) { HIVE_SWITCH_G(g, 6, X) }             \
    else if (mb == 5) { HIVE_SWITCH_G(g, 5, X) }        \
    else if (mb == 4) { HIVE_SWITCH_G(g, 4, X) }        \
    else { HIVE_SWITCH_G(g, 1, X) }

#define HIVE_DISPATCH_GM8(g, mb, X)          \
    if (mb >= 8) {                            \
        switch (g) {                          \
            case 2: X(2, 8); break;           \
            case 4: X(4, 8); break;           \
            default: X(8, 8); break;          \
        }                                     \
    } else if (mb >= 6) {                     \
        switch (g) {                          \
            case 2: X(2, 6); break;           \
            case 4: X(4, 6); break;           \
            default: X(8, 6); break;          \
        }                                     \
    } else {                                  \
        switch (g) {                          \
            case 2: X(2, 1); break;           \
            case 4: X(4, 1); break;           \
            default: X(8, 1); break;          \
        }                                     \
    }

// Byte-wise CRC tables of the §V-B lookup-based pair (reading A-26), written
// to this module's __device__ arrays on the current device.
cudaError_t init_hash_tables() {
    uint32_t t32[256];
    uint64_t t64[256];
    for (uint32_t b = 0; b < 256; ++b) {
        uint32_t c = b;
        uint64_t d = b;
        for (int i = 0; i < 8; ++i) {
            c = (c & 1u) ? (c >> 1) ^ 0xEDB88320u : (c >> 1);
            d = (d & 1ull) ? (d >> 1) ^ 0xC96C5795D7870F42ull : (d >> 1);
        }
        t32[b] = c;
        t64[b] = d;
    }
    cudaError_t e = cudaMemcpyToSymbol(c_crc32_tab, t32, sizeof(t32));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_crc64_tab, t64, sizeof(t64));
    return e;
}

Grids query_grids(int num_sms) {
    Grids g;
    g.g_find = env_g("HIVE_G_FIND", G_FIND);
    g.g_insert = env_g("HIVE_G_INSERT", G_INSERT);
    g.g_slow = env_g("HIVE_G_SLOW", G_SLOW);
    g.g_erase = env_g("HIVE_G_ERASE", G_ERASE);
    g.minb = getenv("HIVE_MINB") ? atoi(getenv("HIVE_MINB")) : MINB_DEFAULT;
    g.minb_find = getenv("HIVE_MINB_FIND") ? atoi(getenv("HIVE_MINB_FIND")) : MINB_FIND_DEFAULT;
    // the Step-3 kernel's residency on its own (experiments; default: as the
    // other mutating kernels)
    g.minb_slow = getenv("HIVE_MINB_SLOW") ? atoi(getenv("HIVE_MINB_SLOW")) : g.minb;
#define OCC_FIND(G, MB) g.find = occ((const void*)k_find<G, MB>) * num_sms
#define OCC_INS(G, MB) g.insert_fast = occ((const void*)k_insert_fast<G, MB>) * num_sms
#define OCC_SLOW(G, MB) g.insert_slow = occ((const void*)k_insert_slow<G, MB>) * num_sms
#define OCC_ERA(G, MB) g.erase = occ((const void*)k_erase<G, MB>) * num_sms
    HIVE_DISPATCH_GM8(g.g_find, g.minb_find, OCC_FIND)
    // HIVE_FIND_BPS: cap the persistent k_find grid at this many blocks per SM
    // (experiments; tools/sector_bench.cu found random 256 B gathers fastest
    // at 4 resident blocks of 256 threads)
    if (getenv("HIVE_FIND_BPS")) g.find = std::min(g.find, atoi(getenv("HIVE_FIND_BPS")) * num_sms);
    HIVE_DISPATCH_GM(g.g_insert, g.minb, OCC_INS)
    HIVE_DISPATCH_GM(g.g_slow, g.minb_slow, OCC_SLOW)
    HIVE_DISPATCH_GM(g.g_erase, g.minb, OCC_ERA)
#define OCC_GATHER(G, MB) g.gather = occ((const void*)k_gather<G, MB>) * num_sms
    HIVE_DISPATCH_GM8(g.g_find, g.minb_find, OCC_GATHER)
    g.dedup = occ((const void*)k_dedup_elect) * num_sms;
    g.stream = 4 * num_sms;
    return g;
}

static inline int clamp_grid(int grid, uint64_t n, uint64_t per_block) {
    uint64_t need = (n + per_block - 1) / per_block;
    if (need < 1) need = 1;
    return (int)(need < (uint64_t)grid ? need : (uint64_t)grid);
}

cudaError_t launch_find(const Grids& gr, cudaStream_t s, const uint32_t* keys, const uint32_t* idx,
                        uint64_t n, const uint64_t* n_dev, TableView tv, StashView sv,
                        uint32_t* vals_out, uint8_t* found, const DupFix* fix) {
    const DupFix fx = fix ? *fix : DupFix{};
    const int grid = (n_dev || fx.flag) ? gr.find : clamp_grid(gr.find, n, BLOCK / gr.g_find);
#define L_FIND(G, MB) k_find<G, MB><<<grid, BLOCK, 0, s>>>(keys, idx, n, n_dev, tv, sv, vals_out, found, fx)
    HIVE_DISPATCH_GM8(gr.g_find, gr.minb_find, L_FIND)
    return cudaGetLastError();
}

cudaError_t launch_dedup_elect_part(int grid, cudaStream_t s, const uint64_t* recs, const uint64_t* part_info,
                                    uint32_t part, DedupView dd, Ctrl* ctrl, uint64_t* clear_next,
                                    uint64_t clear_words) {
    // HIVE_ELECT_ILP: 1 = one record per lane; 2 = two (40 registers, 6 blocks
    // per SM); 3 = two, capped at 32 registers (8 blocks per SM)
    static const int ilp = getenv("HIVE_ELECT_ILP") ? atoi(getenv("HIVE_ELECT_ILP")) : 1;
    static int g2 = 0, g3 = 0;
    int dev = 0, sms = 0;
    if (ilp >= 2 && (!g2 || !g3)) {
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        g2 = occ((const void*)k_dedup_elect_part2<1>) * sms;
        g3 = occ((const void*)k_dedup_elect_part2<8>) * sms;
    }
    if (ilp >= 2 && clear_next) {                 // the two-record variants do not clear
        cudaError_t e = cudaMemsetAsync(clear_next, 0xFF, clear_words * sizeof(uint64_t), s);
        if (e != cudaSuccess) return e;
    }
    if (ilp == 2) k_dedup_elect_part2<1><<<g2, BLOCK, 0, s>>>(recs, part_info, part, dd, ctrl);
    else if (ilp >= 3) k_dedup_elect_part2<8><<<g3, BLOCK, 0, s>>>(recs, part_info, part, dd, ctrl);
    else k_dedup_elect_part<<<grid, BLOCK, 0, s>>>(recs, part_info, part, dd, ctrl,
                                                   reinterpret_cast<uint4*>(clear_next), clear_words / 2);
    return cudaGetLastError();
}

cudaError_t launch_dedup_elect(int grid, cudaStream_t s, const uint32_t* keys, const uint32_t* idx,
                               uint64_t n, const uint64_t* n_dev, DedupView dd, Ctrl* ctrl,
                               const uint32_t* idx2, const uint64_t* n_dev2, const DedupView* dd2) {
    if (!n_dev) grid = clamp_grid(grid, n, BLOCK);
    k_dedup_elect<<<grid, BLOCK, 0, s>>>(keys, idx, n, n_dev, dd, ctrl, idx2, n_dev2, dd2 ? *dd2 : DedupView{});
    return cudaGetLastError();
}

cudaError_t launch_insert_fast(const Grids& gr, cudaStream_t s, const uint32_t* keys, const uint32_t* vals,
                               const uint64_t* kvs, const uint32_t* idx, uint64_t n,
                               const uint64_t* n_dev, TableView tv, StashView sv, DedupView dd,
                               uint8_t* status, uint32_t* vals_zero, uint32_t* leftover,
                               uint32_t op_base, bool prof) {
    const int grid = n_dev ? gr.insert_fast : clamp_grid(gr.insert_fast, n, BLOCK / gr.g_insert);
    if (prof) {                               // step timing: the default geometry only
        k_insert_fast<G_INSERT, MINB_DEFAULT, true><<<grid, BLOCK, 0, s>>>(keys, vals, kvs, idx, n, n_dev, tv, sv,
                                                                           dd, status, vals_zero, leftover, op_base);
        return cudaGetLastError();
    }
#define L_INS(G, MB) k_insert_fast<G, MB><<<grid, BLOCK, 0, s>>>(keys, vals, kvs, idx, n, n_dev, tv, sv, dd, \
                                                         status, vals_zero, leftover, op_base)
    HIVE_DISPATCH_GM(gr.g_insert, gr.minb, L_INS)
    return cudaGetLastError();
}

cudaError_t launch_insert_slow(const Grids& gr, cudaStream_t s, const uint32_t* keys, const uint32_t* vals,
                               const uint64_t* kvs, const uint32_t* leftover, TableView tv,
                               StashView sv, uint32_t max_evictions, uint8_t* status, bool prof) {
    if (prof) {
        k_insert_slow<G_SLOW, MINB_DEFAULT, true><<<gr.insert_slow, BLOCK, 0, s>>>(keys, vals, kvs, leftover, tv, sv,
                                                                                 max_evictions, status);
        return cudaGetLastError();
    }
#define L_SLOW(G, MB) k_insert_slow<G, MB><<<gr.insert_slow, BLOCK, 0, s>>>(keys, vals, kvs, leftover, tv, sv, \
                                                                    max_evictions, status)
    HIVE_DISPATCH_GM(gr.g_slow, gr.minb_slow, L_SLOW)
    return cudaGetLastError();
}

cudaError_t launch_erase(const Grids& gr, cudaStream_t s, const uint32_t* keys, const uint32_t* idx,
                         uint64_t n, const uint64_t* n_dev, TableView tv, StashView sv,
                         DedupView dd, uint8_t* erased, uint32_t* vals_zero, const DupFix* fix) {
    const DupFix fx = fix ? *fix : DupFix{};
    const int grid = (n_dev || fx.flag) ? gr.erase : clamp_grid(gr.erase, n, BLOCK / gr.g_erase);
#define L_ERA(G, MB) k_erase<G, MB><<<grid, BLOCK, 0, s>>>(keys, idx, n, n_dev, tv, sv, dd, erased, vals_zero, fx)
    HIVE_DISPATCH_GM(gr.g_erase, gr.minb, L_ERA)
    return cudaGetLastError();
}

__global__ void __launch_bounds__(BLOCK)
k_count_ops(const uint8_t* __restrict__ ops, uint64_t n, uint8_t code, unsigned long long* __restrict__ out) {
    unsigned long long c = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (uint64_t)gridDim.x * BLOCK)
        c += ops[i] == code;
    block_add(out, c);
}
cudaError_t launch_count_ops(cudaStream_t s, const uint8_t* ops, uint64_t n, uint8_t code,
                             unsigned long long* out) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    k_count_ops<<<clamp_grid(148 * 4, n, BLOCK), BLOCK, 0, s>>>(ops, n, code, out);
    return cudaGetLastError();
}

int mono_grid(int num_sms) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)k_mixed_mono<G_INSERT, G_SLOW>, BLOCK, 0);
    return (nb > 0 ? nb : 1) * num_sms;
}

cudaError_t launch_mixed_mono(int grid, cudaStream_t s, const uint8_t* ops, const uint32_t* keys,
                              const uint32_t* vals, uint64_t n, TableView tv, StashView sv, uint64_t* tab,
                              uint64_t tab_mask, uint8_t* flag, uint32_t* owner_of, uint32_t* leftover,
                              uint32_t max_evictions, uint8_t* result, uint32_t* vals_out) {
    void* args[] = {(void*)&ops, (void*)&keys, (void*)&vals, (void*)&n, (void*)&tv, (void*)&sv, (void*)&tab,
                    (void*)&tab_mask, (void*)&flag, (void*)&owner_of, (void*)&leftover, (void*)&max_evictions,
                    (void*)&result, (void*)&vals_out};
    return cudaLaunchCooperativeKernel((const void*)k_mixed_mono<G_INSERT, G_SLOW>, grid, BLOCK, args, 0, s);
}

// PHASED classification in ONE pass: the op indices of each
// opcode class (0 find, 1 insert, 2 erase) go to region c of out_idx (stride
// `stride`); ops with another opcode get result 0 / value 0 in place.  Each
// tile of CTILE ops reserves its runs with one atomicAdd per class on
// counts[0..2] (zeroed by the caller), so a region is ordered tile by tile in
// reservation order, not in op order: every consumer is order-free (the
// elections keep the highest op index, reading A-15; finds and erases are
// independent per op).  Replaces the count / single-block scan / scatter
// partition for this 3-class case (three launches, ~36 us per 2^20-op batch).
constexpr int CTILE = 4096;
__global__ void __launch_bounds__(BLOCK)
k_classify(const uint8_t* __restrict__ ops, uint64_t n, const uint64_t* __restrict__ n_dev,
           unsigned long long* __restrict__ counts, uint32_t* __restrict__ out_idx, uint64_t stride,
           uint8_t* __restrict__ result_zero, uint32_t* __restrict__ vals_zero) {
    constexpr int PER = CTILE / BLOCK;                   // rows of 32 ops per warp
    __shared__ uint32_t wtot[WARPS_PER_BLOCK][3];
    __shared__ unsigned long long woff[WARPS_PER_BLOCK][3];
    if (n_dev) n = *n_dev;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = lanemask_lt();
    for (uint64_t t0 = (uint64_t)blockIdx.x * CTILE; t0 < n; t0 += (uint64_t)gridDim.x * CTILE) {
        const uint64_t wbase = t0 + (uint64_t)warp * 32 * PER + lane;
        uint32_t cls[PER];
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const uint64_t i = wbase + (uint64_t)r * 32;
            cls[r] = i < n ? (ops[i] < 3 ? ops[i] : 3u) : 4u;
        }
        // per row: rank of the lane inside its class (ballots), running warp totals
        uint32_t c0 = 0, c1 = 0, c2 = 0;
        uint32_t rank[PER];
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const uint32_t b0 = __ballot_sync(FULL, cls[r] == 0), b1 = __ballot_sync(FULL, cls[r] == 1),
                           b2 = __ballot_sync(FULL, cls[r] == 2);
            const uint32_t bm = cls[r] == 0 ? b0 : cls[r] == 1 ? b1 : b2;
            const uint32_t run = cls[r] == 0 ? c0 : cls[r] == 1 ? c1 : c2;
            rank[r] = run + __popc(bm & lt);
            c0 += __popc(b0);
            c1 += __popc(b1);
            c2 += __popc(b2);
        }
        if (lane == 0) {
            wtot[warp][0] = c0;
            wtot[warp][1] = c1;
            wtot[warp][2] = c2;
        }
        __syncthreads();
        if (threadIdx.x < 3) {                            // one reservation per class per tile
            const int c = threadIdx.x;
            uint32_t tot = 0;
            for (int w = 0; w < WARPS_PER_BLOCK; ++w) tot += wtot[w][c];
            unsigned long long base = tot ? atomicAdd(&counts[c], (unsigned long long)tot) : 0ull;
            for (int w = 0; w < WARPS_PER_BLOCK; ++w) {
                woff[w][c] = base;
                base += wtot[w][c];
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const uint64_t i = wbase + (uint64_t)r * 32;
            if (cls[r] < 3) {
                out_idx[cls[r] * stride + woff[warp][cls[r]] + rank[r]] = (uint32_t)i;
            } else if (cls[r] == 3) {
                if (result_zero) result_zero[i] = 0;
                if (vals_zero) vals_zero[i] = 0;
            }
        }
        __syncthreads();                                  // wtot / woff reuse
    }
}
// Per-batch scratch reset of hive_mixed in ONE launch (each cudaMemsetAsync
// on this path cost a few microseconds of GPU time per batch): the class
// counts, the Step-3 list cursor pair, the paired election's flags (zero) and
// sub-tables (all ones).  fbytes and dwords are multiples of 16 and 2.
__global__ void __launch_bounds__(BLOCK)
k_batch_prep(Ctrl* ctrl, int zero_left, uint4* __restrict__ flag, uint64_t f16, uint4* __restrict__ dd, uint64_t d16) {
    const uint64_t tid = (uint64_t)blockIdx.x * BLOCK + threadIdx.x, stride = (uint64_t)gridDim.x * BLOCK;
    if (tid == 0) {
        ctrl->cls_n[0] = ctrl->cls_n[1] = ctrl->cls_n[2] = 0;
        if (zero_left) ctrl->n_left = ctrl->slow_next = 0;
    }
    const uint4 z = make_uint4(0u, 0u, 0u, 0u), o = make_uint4(~0u, ~0u, ~0u, ~0u);
    for (uint64_t i = tid; i < f16; i += stride) flag[i] = z;
    for (uint64_t i = tid; i < d16; i += stride) dd[i] = o;
}
cudaError_t launch_batch_prep(cudaStream_t s, Ctrl* ctrl, bool zero_left, uint8_t* flag, uint64_t fbytes,
                              uint64_t* dd, uint64_t dwords, int num_sms) {
    const uint64_t work = std::max<uint64_t>(fbytes / 16, dwords / 2);
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((work + BLOCK - 1) / BLOCK, (uint64_t)num_sms * 8));
    k_batch_prep<<<grid, BLOCK, 0, s>>>(ctrl, zero_left ? 1 : 0, reinterpret_cast<uint4*>(flag), fbytes / 16,
                                        reinterpret_cast<uint4*>(dd), dwords / 2);
    return cudaGetLastError();
}

cudaError_t launch_classify(cudaStream_t s, const uint8_t* ops, uint64_t n, const uint64_t* n_dev,
                            uint64_t* counts, uint32_t* out_idx, uint64_t stride, uint8_t* result_zero,
                            uint32_t* vals_zero, int num_sms, bool counts_zeroed) {
    cudaError_t e = counts_zeroed ? cudaSuccess : cudaMemsetAsync(counts, 0, 3 * sizeof(uint64_t), s);
    if (e != cudaSuccess || n == 0) return e;
    const int grid = (int)std::min<uint64_t>((n + CTILE - 1) / CTILE, (uint64_t)num_sms * 8);
    k_classify<<<grid, BLOCK, 0, s>>>(ops, n, n_dev, reinterpret_cast<unsigned long long*>(counts), out_idx, stride,
                                      result_zero, vals_zero);
    return cudaGetLastError();
}

cudaError_t launch_dup_copy(int grid, cudaStream_t s, const uint32_t* idx, uint64_t n,
                            const uint64_t* n_dev, DedupView dd, uint8_t* out) {
    if (!n_dev) grid = clamp_grid(grid, n, BLOCK);
    k_dup_copy<<<grid, BLOCK, 0, s>>>(idx, n, n_dev, dd, out);
    return cudaGetLastError();
}

cudaError_t launch_split(cudaStream_t s, TableView tv, uint32_t n_pairs, Ctrl* ctrl) {
    if (n_pairs == 0) return cudaSuccess;
    const int grid = (int)((n_pairs + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK);
    k_split<<<grid, BLOCK, 0, s>>>(tv, n_pairs, ctrl);
    return cudaGetLastError();
}

cudaError_t launch_merge(cudaStream_t s, TableView tv, uint32_t n_pairs, unsigned long long* abort_at,
                         const unsigned long long* prev_abort, uint64_t prev_pairs) {
    if (n_pairs == 0) return cudaSuccess;
    const int grid = (int)((n_pairs + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK);
    k_merge_check<<<grid, BLOCK, 0, s>>>(tv, n_pairs, abort_at, prev_abort, prev_pairs);
    k_merge_apply<<<grid, BLOCK, 0, s>>>(tv, n_pairs, abort_at);
    return cudaGetLastError();
}

cudaError_t launch_dump(int grid, cudaStream_t s, TableView tv, uint64_t n_buckets, StashView sv,
                        uint32_t* keys, uint32_t* vals, uint64_t cap) {
    const uint64_t ring_n = sv.cap;
    k_dump<<<grid, BLOCK, 0, s>>>(tv, n_buckets * SLOTS, sv, ring_n, keys, vals, cap);
    return cudaGetLastError();
}

cudaError_t launch_count_b1(int grid, cudaStream_t s, TableView tv, uint64_t n_buckets, Ctrl* ctrl) {
    k_count_b1<<<grid, BLOCK, 0, s>>>(tv, n_buckets * SLOTS, ctrl);
    return cudaGetLastError();
}

// Elements per warp of the stable partition: enough warps to fill the GPU for
// small batches (a 2^20-op classify ran on 512 warps at 2048 per warp),
// PART_CHUNK for large ones (bounds the single-block scan).
uint32_t part_chunk(uint64_t n) {
    uint64_t c = 256;
    while (c < (uint64_t)PART_CHUNK && c * 16384 < n) c *= 2;
    return (uint32_t)c;
}
uint64_t part_warps(uint64_t n) { const uint64_t c = part_chunk(n); return (n + c - 1) / c; }

cudaError_t launch_partition_pd(cudaStream_t s, int mode, uint32_t n_parts, uint32_t seed,
                                const uint32_t* keys, const uint32_t* vals, const uint8_t* ops,
                                uint64_t n, uint64_t* cnt, uint64_t* part_info, uint64_t* send_kv,
                                uint8_t* send_ops, uint32_t* pos, const uint32_t* idx, const uint64_t* n_dev,
                                const PeerDest& pd);

cudaError_t launch_partition(cudaStream_t s, int mode, uint32_t n_parts, uint32_t seed,
                             const uint32_t* keys, const uint32_t* vals, const uint8_t* ops,
                             uint64_t n, uint64_t* cnt, uint64_t* part_info, uint64_t* send_kv,
                             uint8_t* send_ops, uint32_t* pos, const uint32_t* idx, const uint64_t* n_dev) {
    return launch_partition_pd(s, mode, n_parts, seed, keys, vals, ops, n, cnt, part_info, send_kv, send_ops, pos,
                               idx, n_dev, PeerDest{});
}

cudaError_t launch_partition_pd(cudaStream_t s, int mode, uint32_t n_parts, uint32_t seed,
                                const uint32_t* keys, const uint32_t* vals, const uint8_t* ops,
                                uint64_t n, uint64_t* cnt, uint64_t* part_info, uint64_t* send_kv,
                                uint8_t* send_ops, uint32_t* pos, const uint32_t* idx, const uint64_t* n_dev,
                                const PeerDest& pd) {
    const uint64_t nw = part_warps(n);
    const uint32_t chunk = part_chunk(n);
    const int grid = (int)((nw + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK);
    if (nw) k_part_count<<<grid, BLOCK, 0, s>>>(mode, n_parts, seed, keys, ops, n, nw, cnt, idx, n_dev, chunk);
    k_part_scan<<<1, 1024, 0, s>>>(cnt, (uint64_t)n_parts * nw, n_parts, nw, part_info);
    if (nw)
        k_part_scatter<<<grid, BLOCK, 0, s>>>(mode, n_parts, seed, keys, vals, ops, n, nw, cnt, part_info,
                                              send_kv, send_ops, pos, idx, n_dev, chunk, pd);
    return cudaGetLastError();
}

cudaError_t launch_unroute(cudaStream_t s, const uint32_t* pos, uint64_t n, const uint8_t* in8,
                           uint8_t* out8, const uint32_t* in32, uint32_t* out32) {
    const int grid = clamp_grid(1184, n, BLOCK);
    k_unroute<<<grid, BLOCK, 0, s>>>(pos, n, in8, out8, in32, out32);
    return cudaGetLastError();
}

// ---- sharded table over NCCL: padded exchange ------------------------------------
__global__ void k_pad_counts(const uint64_t* __restrict__ part_info, uint32_t n_shards, uint64_t cap,
                             uint64_t* __restrict__ cnt_send, Ctrl* ctrl) {
    const uint32_t p = threadIdx.x;
    unsigned long long over = 0;
    if (p < n_shards) {
        const uint64_t c = part_info[p];
        cnt_send[p] = c < cap ? c : cap;
        over = c > cap ? c - cap : 0;
    }
    over = warp_sum(over);                      // n_shards <= 32 (one warp)
    if (p == 0 && over) atomicAdd(&ctrl->xfail, over);
}

// Region prefix of the n_src clipped counts, per block (n_src <= MAX_PARTS).
__device__ __forceinline__ void pad_starts(const uint64_t* cnt, uint32_t n_src, uint64_t cap, uint64_t* start) {
    if (threadIdx.x == 0) {
        uint64_t a = 0;
        for (uint32_t r = 0; r < n_src; ++r) {
            start[r] = a;
            a += cnt[r] < cap ? cnt[r] : cap;
        }
        start[n_src] = a;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(BLOCK)
k_owner_compact(uint32_t n_src, uint64_t cap, const uint64_t* __restrict__ recv_kv,
                const uint8_t* __restrict__ recv_ops, const uint64_t* __restrict__ cnt,
                uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, uint8_t* __restrict__ ops,
                uint32_t* __restrict__ back, uint64_t* __restrict__ n_dev, uint32_t self,
                const uint64_t* __restrict__ self_kv, const uint8_t* __restrict__ self_ops) {
    __shared__ uint64_t start[MAX_PARTS + 1];
    pad_starts(cnt, n_src, cap, start);
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_dev = start[n_src];
    const uint64_t total = (uint64_t)n_src * cap;
    for (uint64_t j = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; j < total; j += (uint64_t)gridDim.x * BLOCK) {
        const uint32_t r = (uint32_t)(j / cap);
        const uint64_t o = j - (uint64_t)r * cap;
        if (start[r] + o >= start[r + 1]) continue;          // padding
        const uint64_t li = start[r] + o;
        // this rank's own region never went through the exchange: it is read
        // from the send buffer (same padded layout)
        const bool own = self_kv && r == self;
        const uint64_t w = own ? self_kv[j] : recv_kv[j];
        keys[li] = key_of(w);
        vals[li] = val_of(w);
        if (ops) ops[li] = own ? self_ops[j] : recv_ops[j];
        back[li] = (uint32_t)j;
    }
}

__global__ void __launch_bounds__(BLOCK)
k_owner_return(uint64_t n, const uint64_t* __restrict__ n_dev, const uint32_t* __restrict__ back,
               const uint8_t* __restrict__ r8, const uint32_t* __restrict__ r32, uint8_t* __restrict__ ret8,
               uint32_t* __restrict__ ret32) {
    if (n_dev) n = *n_dev;
    for (uint64_t j = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; j < n; j += (uint64_t)gridDim.x * BLOCK) {
        const uint32_t at = back[j];
        if (r8) ret8[at] = r8[j];
        if (r32) ret32[at] = r32[j];
    }
}

__global__ void __launch_bounds__(BLOCK)
k_unroute_pad(const uint32_t* __restrict__ pos, uint64_t n, const uint8_t* __restrict__ in8,
              uint8_t* __restrict__ out8, const uint32_t* __restrict__ in32, uint32_t* __restrict__ out32,
              uint8_t miss8, const unsigned long long* __restrict__ poison, const uint32_t* __restrict__ idx,
              const uint64_t* __restrict__ n_dev) {
    // a set poison word (peer-exchange timeout marker): no result is trusted
    const bool lost = poison && *(volatile const unsigned long long*)poison != 0;
    if (n_dev) n = *n_dev;
    for (uint64_t i = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (uint64_t)gridDim.x * BLOCK) {
        const uint32_t p = pos[i];
        const bool ok = p != NO_POS && !lost;
        const uint64_t o = idx ? idx[i] : i;          // index-list route: results go to op idx[i]
        if (out8) out8[o] = ok ? in8[p] : (lost ? HIVE_RESULT_PEER_LOST : miss8);
        if (out32) out32[o] = ok ? in32[p] : 0u;
    }
}

// ---- source-side owner election of a sharded call (SURVEY §8(e) Zipf item) -------
// Group of an op = (key, class); class = the op's opcode (0 find, 1 insert,
// 2 erase; other opcodes and the reserved key are never grouped).  The highest
// op index of a group is its owner; only owners are routed, the others copy
// their owner's result after the exchange.  Same results as routing every op:
// the owner's batch is PHASED and a rank's duplicates are consecutive members
// of the union batch's groups.
__device__ __forceinline__ uint32_t src_hash(uint32_t k, uint32_t cls) {
    return fmix32(k ^ DEDUP_SEED ^ (cls * 0x9E3779B9u));
}
__global__ void __launch_bounds__(BLOCK)
k_src_elect(const uint8_t* __restrict__ opc, uint8_t kind_op, const uint32_t* __restrict__ keys, uint64_t n,
            uint64_t* __restrict__ tab, uint64_t mask, uint8_t* __restrict__ flag, Ctrl* ctrl) {
    const int lane = threadIdx.x & 31;
    for (uint64_t t0 = ((uint64_t)blockIdx.x * BLOCK + threadIdx.x) & ~31ull; t0 < n;
         t0 += (uint64_t)gridDim.x * BLOCK) {
        const uint64_t t = t0 + lane;
        const uint32_t o = t < n ? (opc ? opc[t] : kind_op) : 3u;
        const uint32_t k = t < n ? keys[t] : INVALID_KEY;
        const bool part = o < 3 && k != INVALID_KEY;
        const uint32_t grp = __match_any_sync(FULL, part ? ((uint64_t)k << 2 | o) : ~0ull);
        if (!part) continue;
        if (__popc(grp) > 1) flag[t] = 1;
        if ((31 - __clz(grp)) != lane) continue;                 // warp pre-merge: the max lane
        const uint64_t word = ((uint64_t)k << 32) | ((uint64_t)o << 30) | (uint32_t)t;
        uint64_t h = src_hash(k, o) & mask;
        uint64_t probe = 0;
        for (; probe <= mask; ++probe) {
            const uint64_t prev = cas64(&tab[h], EMPTY, word);
            if (prev == EMPTY) break;
            if ((prev >> 30) == (word >> 30)) {                   // same key and class
                flag[t] = 1;
                flag[(uint32_t)prev & 0x3FFFFFFFu] = 1;
                if (word > prev) atomicMax((unsigned long long*)&tab[h], (unsigned long long)word);
                break;
            }
            h = (h + 1) & mask;
        }
        if (probe > mask) atomicAdd(&ctrl->eover, 1ull);
    }
}
// The send list (owners and ungrouped ops, in no particular order) and, for
// grouped ops, their owner.
__global__ void __launch_bounds__(BLOCK)
k_src_list(const uint8_t* __restrict__ opc, uint8_t kind_op, const uint32_t* __restrict__ keys, uint64_t n,
           const uint64_t* __restrict__ tab, uint64_t mask, const uint8_t* __restrict__ flag,
           uint32_t* __restrict__ owner_of, uint32_t* __restrict__ list, unsigned long long* __restrict__ n_list) {
    const int lane = threadIdx.x & 31;
    for (uint64_t t0 = ((uint64_t)blockIdx.x * BLOCK + threadIdx.x) & ~31ull; t0 < n;
         t0 += (uint64_t)gridDim.x * BLOCK) {
        const uint64_t t = t0 + lane;
        bool send = t < n;
        if (send && flag[t]) {
            const uint32_t o = opc ? opc[t] : kind_op, k = keys[t];
            uint64_t h = src_hash(k, o) & mask;
            uint32_t own = (uint32_t)t;
            for (uint64_t probe = 0; probe <= mask; ++probe) {
                const uint64_t e = tab[h];
                if (e == EMPTY) break;
                if ((e >> 32) == k && ((e >> 30) & 3u) == o) { own = (uint32_t)e & 0x3FFFFFFFu; break; }
                h = (h + 1) & mask;
            }
            owner_of[t] = own;
            send = own == (uint32_t)t;
        }
        const uint32_t bal = __ballot_sync(FULL, send);
        unsigned long long base = 0;
        if (lane == 0 && bal) base = atomicAdd(n_list, (unsigned long long)__popc(bal));
        base = __shfl_sync(FULL, base, 0);
        if (send) list[base + __popc(bal & lanemask_lt())] = (uint32_t)t;
    }
}
__global__ void __launch_bounds__(BLOCK)
k_src_copy(uint64_t n, const uint8_t* __restrict__ flag, const uint32_t* __restrict__ owner_of,
           uint8_t* __restrict__ out8, uint32_t* __restrict__ out32) {
    for (uint64_t t = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; t < n; t += (uint64_t)gridDim.x * BLOCK) {
        if (!flag[t]) continue;
        const uint32_t o = owner_of[t];
        if (o == (uint32_t)t) continue;
        if (out8) out8[t] = out8[o];
        if (out32) out32[t] = out32[o];
    }
}
cudaError_t launch_src_elect(cudaStream_t s, const uint8_t* opc, uint8_t kind_op, const uint32_t* keys, uint64_t n,
                             uint64_t* tab, uint64_t mask, uint8_t* flag, uint32_t* owner_of, uint32_t* list,
                             unsigned long long* n_list, Ctrl* ctrl) {
    cudaError_t e = cudaMemsetAsync(tab, 0xFF, (mask + 1) * sizeof(uint64_t), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(flag, 0, n, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(n_list, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    const int grid = clamp_grid(148 * 8, n, BLOCK);
    k_src_elect<<<grid, BLOCK, 0, s>>>(opc, kind_op, keys, n, tab, mask, flag, ctrl);
    k_src_list<<<grid, BLOCK, 0, s>>>(opc, kind_op, keys, n, tab, mask, flag, owner_of, list, n_list);
    return cudaGetLastError();
}
cudaError_t launch_src_copy(cudaStream_t s, uint64_t n, const uint8_t* flag, const uint32_t* owner_of, uint8_t* out8,
                            uint32_t* out32) {
    if (n == 0) return cudaSuccess;
    k_src_copy<<<clamp_grid(148 * 8, n, BLOCK), BLOCK, 0, s>>>(n, flag, owner_of, out8, out32);
    return cudaGetLastError();
}

cudaError_t launch_route_pad(cudaStream_t s, uint32_t n_shards, uint32_t seed, const uint32_t* keys,
                             const uint32_t* vals, const uint8_t* ops, uint64_t n, uint64_t cap, uint64_t* cnt,
                             uint64_t* part_info, uint64_t* send_kv, uint8_t* send_ops, uint32_t* pos,
                             uint64_t* cnt_send, Ctrl* ctrl, const uint32_t* idx, const uint64_t* n_dev) {
    PeerDest pd{};
    pd.region = cap;
    cudaError_t e = launch_partition_pd(s, PART_ROUTE_PAD, n_shards, seed, keys, vals, ops, n, cnt, part_info,
                                        send_kv, send_ops, pos, idx, n_dev, pd);
    if (e != cudaSuccess) return e;
    k_pad_counts<<<1, 32, 0, s>>>(part_info, n_shards, cap, cnt_send, ctrl);
    return cudaGetLastError();
}

cudaError_t launch_owner_compact(cudaStream_t s, uint32_t n_src, uint64_t cap, const uint64_t* recv_kv,
                                 const uint8_t* recv_ops, const uint64_t* cnt_recv, uint32_t* keys, uint32_t* vals,
                                 uint8_t* ops, uint32_t* back, uint64_t* n_dev, uint32_t self,
                                 const uint64_t* self_kv, const uint8_t* self_ops) {
    const int grid = clamp_grid(148 * 8, (uint64_t)n_src * cap, BLOCK);
    k_owner_compact<<<grid, BLOCK, 0, s>>>(n_src, cap, recv_kv, recv_ops, cnt_recv, keys, vals, ops, back, n_dev,
                                           self, self_kv, self_ops);
    return cudaGetLastError();
}

cudaError_t launch_owner_return(cudaStream_t s, uint64_t n_upper, const uint64_t* n_dev, const uint32_t* back,
                                const uint8_t* r8, const uint32_t* r32, uint8_t* ret8, uint32_t* ret32) {
    const int grid = clamp_grid(148 * 8, n_upper, BLOCK);
    k_owner_return<<<grid, BLOCK, 0, s>>>(n_upper, n_dev, back, r8, r32, ret8, ret32);
    return cudaGetLastError();
}

cudaError_t launch_unroute_pad(cudaStream_t s, const uint32_t* pos, uint64_t n, const uint8_t* in8, uint8_t* out8,
                               const uint32_t* in32, uint32_t* out32, uint8_t miss8,
                               const unsigned long long* poison, const uint32_t* idx, const uint64_t* n_dev) {
    if (n == 0) return cudaSuccess;
    const int grid = clamp_grid(148 * 8, n, BLOCK);
    k_unroute_pad<<<grid, BLOCK, 0, s>>>(pos, n, in8, out8, in32, out32, miss8, poison, idx, n_dev);
    return cudaGetLastError();
}

// ---- test hook: load an externally built image (hive_load_image) -----------------
// Spill words of a loaded bucket array: every key not in bucket addr(h1(k))
// sets its fingerprint bits there; stash entries are written to the ring,
// indexed, and flagged in their b1's spill word the same way.
__global__ void __launch_bounds__(BLOCK)
k_image_spill(TableView tv, uint64_t n_slots) {
    for (uint64_t i = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; i < n_slots; i += (uint64_t)gridDim.x * BLOCK) {
        const uint64_t w = tv.buckets[i];
        if (w == EMPTY) continue;
        const uint32_t k = key_of(w), hb = tv.addr(tv.h1(k));
        if (hb != (uint32_t)(i / SLOTS)) atomicOr((unsigned long long*)&tv.spill[hb], (unsigned long long)spill_fp(k));
    }
}
__global__ void __launch_bounds__(BLOCK)
k_image_stash(TableView tv, StashView sv, const uint64_t* __restrict__ words, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (uint64_t)gridDim.x * BLOCK) {
        const uint64_t w = words[i];
        const uint32_t k = key_of(w);
        sv.ring[i] = w;
        stash_index_put(sv, k, i);
        atomicOr((unsigned long long*)&tv.spill[tv.addr(tv.h1(k))], (unsigned long long)spill_fp(k));
    }
}
cudaError_t launch_image(cudaStream_t s, TableView tv, uint64_t n_buckets, StashView sv, const uint64_t* stash,
                         uint64_t n_stash) {
    k_image_spill<<<clamp_grid(148 * 8, n_buckets * SLOTS, BLOCK), BLOCK, 0, s>>>(tv, n_buckets * SLOTS);
    if (n_stash) k_image_stash<<<clamp_grid(148 * 8, n_stash, BLOCK), BLOCK, 0, s>>>(tv, sv, stash, n_stash);
    return cudaGetLastError();
}

// ---- hash study (§III-C, Theorem 1 / CSR; §V-B pairs) -------------------------
__device__ __forceinline__ uint32_t hash_fn(uint32_t fn, uint32_t k) {
    switch (fn) {
        case 0: return bithash1(k);
        case 1: return bithash2(k);
        case 2: return crc32_key(k);
        default: return crc64_key(k);
    }
}
__global__ void __launch_bounds__(BLOCK)
k_hash(uint32_t fn, const uint32_t* __restrict__ keys, uint64_t n, uint32_t* __restrict__ out,
       uint32_t* __restrict__ bins, uint64_t m) {
    for (uint64_t i = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; i < n; i += (uint64_t)gridDim.x * BLOCK) {
        const uint32_t h = hash_fn(fn, keys[i]);
        if (out) out[i] = h;
        if (bins) {                       // occupancy bitmap of bin = h mod m
            const uint64_t b = h % m;
            atomicOr(&bins[b >> 5], 1u << (b & 31));
        }
    }
}
__global__ void __launch_bounds__(BLOCK)
k_popc(const uint32_t* __restrict__ bins, uint64_t words, unsigned long long* __restrict__ total) {
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; i < words; i += (uint64_t)gridDim.x * BLOCK)
        c += __popc(bins[i]);
    c = __reduce_add_sync(0xFFFFFFFFu, (unsigned)c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(total, c);
}
cudaError_t launch_hash(cudaStream_t s, uint32_t fn, const uint32_t* keys, uint64_t n, uint32_t* out,
                        uint32_t* bins, uint64_t m) {
    const int grid = (int)std::min<uint64_t>((n + BLOCK - 1) / BLOCK, 148ull * 16);
    k_hash<<<grid, BLOCK, 0, s>>>(fn, keys, n, out, bins, m);
    return cudaGetLastError();
}
cudaError_t launch_popc(cudaStream_t s, const uint32_t* bins, uint64_t words, unsigned long long* total) {
    const int grid = (int)std::min<uint64_t>((words + BLOCK - 1) / BLOCK, 148ull * 16);
    k_popc<<<grid > 0 ? grid : 1, BLOCK, 0, s>>>(bins, words, total);
    return cudaGetLastError();
}

cudaError_t launch_gather(const Grids& gr, cudaStream_t s, const uint32_t* keys, uint64_t n,
                          const uint64_t* blocks, uint64_t n_blocks, uint32_t* out, uint32_t mode) {
    const int grid = clamp_grid(gr.gather, n, BLOCK / gr.g_find);
#define L_GATHER(G, MB) k_gather<G, MB><<<grid, BLOCK, 0, s>>>(keys, n, blocks, n_blocks, out, mode)
    HIVE_DISPATCH_GM8(gr.g_find, gr.minb_find, L_GATHER)
    return cudaGetLastError();
}

cudaError_t launch_unpack(cudaStream_t s, const uint64_t* kv, uint64_t n, uint32_t* keys,
                          uint32_t* vals) {
    const int grid = clamp_grid(1184, n, BLOCK);
    k_unpack<<<grid, BLOCK, 0, s>>>(kv, n, keys, vals);
    return cudaGetLastError();
}

// Two word ranges set to EMPTY in one launch (the growth of a clean stash:
// only the newly exposed ring and index words).
__global__ void __launch_bounds__(BLOCK)
k_fill2(uint64_t* __restrict__ a, uint64_t na, uint64_t* __restrict__ b, uint64_t nb) {
    const uint64_t stride = (uint64_t)gridDim.x * BLOCK;
    for (uint64_t i = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; i < na + nb; i += stride) {
        if (i < na) a[i] = EMPTY;
        else b[i - na] = EMPTY;
    }
}
cudaError_t launch_fill2(cudaStream_t s, uint64_t* a, uint64_t na, uint64_t* b, uint64_t nb, int num_sms) {
    if (na + nb == 0) return cudaSuccess;
    const int grid = (int)std::min<uint64_t>((na + nb + BLOCK - 1) / BLOCK, (uint64_t)num_sms * 4);
    k_fill2<<<grid, BLOCK, 0, s>>>(a, na, b, nb);
    return cudaGetLastError();
}

cudaError_t launch_stash_reset(cudaStream_t s, StashView sv) {
    cudaError_t e = cudaMemsetAsync(sv.ring, 0xFF, sv.cap * sizeof(uint64_t), s);
    if (e != cudaSuccess) return e;
    return cudaMemsetAsync(sv.index, 0xFF, (sv.idx_mask + 1) * sizeof(uint64_t), s);
}

// ---- NEXT-1 peer-memory exchange -------------------------------------
// Per-source count of this rank's records, written into every owner's count
// array (remote stores), after the scatter in stream order.
__global__ void k_p2p_counts(const uint64_t* __restrict__ part_info, uint32_t n_shards, PeerDest pd,
                             unsigned long long* xfail) {
    const uint32_t p = threadIdx.x;
    unsigned long long over = 0;
    if (p < n_shards) {
        const uint64_t c = part_info[p];
        pd.cnt[p][pd.rank] = c < pd.region ? c : pd.region;       // records actually stored
        over = c > pd.region ? c - pd.region : 0;
    }
    over = warp_sum(over);
    if (p == 0 && over && xfail) atomicAdd(xfail, over);
    __threadfence_system();
}

// Owner, device-count form: result j of the compacted inbox batch goes back to
// the source region its record came from (back[j] = source * region + slot).
__global__ void __launch_bounds__(BLOCK)
k_return_p2p_back(const uint64_t* __restrict__ n_dev, uint64_t region, const uint32_t* __restrict__ back,
                  const uint32_t* __restrict__ res32, const uint8_t* __restrict__ res8, PeerDest pd) {
    const uint64_t n = *n_dev;
    for (uint64_t j = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; j < n; j += (uint64_t)gridDim.x * BLOCK) {
        const uint32_t at = back[j];
        const uint32_t r = (uint32_t)(at / region);
        const uint64_t dst = (uint64_t)pd.rank * region + (at - (uint64_t)r * region);
        if (res32) pd.res32[r][dst] = res32[j];
        if (res8) pd.res8[r][dst] = res8[j];
    }
    __threadfence_system();
}
cudaError_t launch_return_p2p_back(cudaStream_t s, uint64_t n_upper, const uint64_t* n_dev, uint64_t region,
                                   const uint32_t* back, const uint32_t* res32, const uint8_t* res8,
                                   const PeerDest& pd) {
    const int grid = clamp_grid(148 * 8, n_upper, BLOCK);
    k_return_p2p_back<<<grid, BLOCK, 0, s>>>(n_dev, region, back, res32, res8, pd);
    return cudaGetLastError();
}

// Region prefix of the n_src per-source counts (n_src <= MAX_PEERS), per block.
__device__ __forceinline__ void region_starts(const uint64_t* cnt, uint32_t n_src, uint64_t* start) {
    if (threadIdx.x == 0) {
        uint64_t a = 0;
        for (uint32_t r = 0; r < n_src; ++r) {
            start[r] = a;
            a += cnt[r];
        }
        start[n_src] = a;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(BLOCK)
k_inbox_compact(uint32_t n_src, uint64_t region, const uint64_t* __restrict__ inbox_kv,
                const uint8_t* __restrict__ inbox_ops, const uint64_t* __restrict__ cnt, uint64_t n_total,
                uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, uint8_t* __restrict__ ops) {
    __shared__ uint64_t start[MAX_PEERS + 1];
    region_starts(cnt, n_src, start);
    for (uint64_t j = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; j < n_total; j += (uint64_t)gridDim.x * BLOCK) {
        uint32_t r = 0;
        while (r + 1 < n_src && start[r + 1] <= j) ++r;
        const uint64_t at = (uint64_t)r * region + (j - start[r]);
        const uint64_t w = inbox_kv[at];
        keys[j] = key_of(w);
        vals[j] = val_of(w);
        if (ops) ops[j] = inbox_ops[at];
    }
}

__global__ void __launch_bounds__(BLOCK)
k_return_p2p(uint32_t n_src, const uint64_t* __restrict__ cnt, uint64_t n_total,
             const uint32_t* __restrict__ res32, const uint8_t* __restrict__ res8, PeerDest pd) {
    __shared__ uint64_t start[MAX_PEERS + 1];
    region_starts(cnt, n_src, start);
    for (uint64_t j = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; j < n_total; j += (uint64_t)gridDim.x * BLOCK) {
        uint32_t r = 0;
        while (r + 1 < n_src && start[r + 1] <= j) ++r;
        // source r's result region of this owner (remote store)
        const uint64_t at = (uint64_t)pd.rank * pd.region + (j - start[r]);
        if (res32) pd.res32[r][at] = res32[j];
        if (res8) pd.res8[r][at] = res8[j];
    }
    __threadfence_system();
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_p2p_signal(uint32_t n, uint32_t phase, uint64_t epoch, PeerDest pd) {
    const uint32_t p = threadIdx.x;
    __threadfence_system();                       // this rank's earlier stores first
    if (p < n) {
        unsigned long long* w = pd.sig[p] + phase * MAX_PEERS + pd.rank;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(w), "l"((unsigned long long)epoch) : "memory");
    }
}

__global__ void k_p2p_wait(uint32_t n, uint32_t phase, uint64_t epoch, unsigned long long* sig_own,
                           uint64_t timeout_ns) {
    const uint32_t r = threadIdx.x;
    if (r < n) {
        const unsigned long long* w = sig_own + phase * MAX_PEERS + r;
        const uint64_t t0 = globaltimer();
        while (true) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(w) : "memory");
            if (v >= epoch) break;
            if (globaltimer() - t0 > timeout_ns) {          // a peer never arrived: flag, do not hang
                atomicExch(sig_own + 2 * MAX_PEERS, 1ull);
                break;
            }
            __nanosleep(200);
        }
    }
    __threadfence_system();
}

cudaError_t launch_p2p_signal(cudaStream_t s, uint32_t n, uint32_t phase, uint64_t epoch, const PeerDest& pd) {
    k_p2p_signal<<<1, 32, 0, s>>>(n, phase, epoch, pd);
    return cudaGetLastError();
}

cudaError_t launch_p2p_wait(cudaStream_t s, uint32_t n, uint32_t phase, uint64_t epoch,
                            unsigned long long* sig_own, uint64_t timeout_ns) {
    k_p2p_wait<<<1, 32, 0, s>>>(n, phase, epoch, sig_own, timeout_ns);
    return cudaGetLastError();
}

cudaError_t launch_route_p2p(cudaStream_t s, uint32_t n_shards, uint32_t seed, const uint32_t* keys,
                             const uint32_t* vals, const uint8_t* ops, uint64_t n, uint64_t* cnt,
                             uint64_t* part_info, uint32_t* pos, const PeerDest& pd, unsigned long long* xfail) {
    cudaError_t e = launch_partition_pd(s, PART_ROUTE_P2P, n_shards, seed, keys, vals, ops, n, cnt, part_info,
                                        nullptr, nullptr, pos, nullptr, nullptr, pd);
    if (e != cudaSuccess) return e;
    k_p2p_counts<<<1, 32, 0, s>>>(part_info, n_shards, pd, xfail);
    return cudaGetLastError();
}

cudaError_t launch_inbox_compact(cudaStream_t s, uint32_t n_src, uint64_t region, const uint64_t* inbox_kv,
                                 const uint8_t* inbox_ops, const uint64_t* cnt, uint64_t n_total,
                                 uint32_t* keys, uint32_t* vals, uint8_t* ops) {
    if (!n_total) return cudaSuccess;
    const int grid = clamp_grid(148 * 8, n_total, BLOCK);
    k_inbox_compact<<<grid, BLOCK, 0, s>>>(n_src, region, inbox_kv, inbox_ops, cnt, n_total, keys, vals, ops);
    return cudaGetLastError();
}

cudaError_t launch_return_p2p(cudaStream_t s, uint32_t n_src, const uint64_t* cnt, uint64_t n_total,
                              const uint32_t* res32, const uint8_t* res8, const PeerDest& pd) {
    if (!n_total) return cudaSuccess;
    const int grid = clamp_grid(148 * 8, n_total, BLOCK);
    k_return_p2p<<<grid, BLOCK, 0, s>>>(n_src, cnt, n_total, res32, res8, pd);
    return cudaGetLastError();
}

}  // namespace hive
