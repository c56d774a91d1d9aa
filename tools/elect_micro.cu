// Micro-benchmark for the owner election: where do the
// 46 us per 2^21-op part go, and what would a bitmap pre-filter cost?
//   E1  part election as in k_dedup_elect_part (MATCH.ANY + CAS64 on a
//       freshly memset 64 MiB sub-table), memset and kernel timed apart
//   E2  the same without MATCH.ANY
//   E3  the same run twice on the same (already L2-resident) sub-table
//   E4  bitmap pre-filter over a whole 2^26-op phase: atomicOr-with-return
//       into a B-bit "seen" map, RED.OR into a "dup" map; then a read pass
//       counting the flagged ops (false positives at B = 2^28 / 2^29 / 2^30)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/elect_micro tools/elect_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define FULL 0xffffffffu
constexpr uint64_t EMPTY = ~0ull;

__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
    h ^= h >> 16; h *= 0x85ebca6bu; h ^= h >> 13; h *= 0xc2b2ae35u; h ^= h >> 16; return h;
}

// records (op << 32 | key) of one part
__global__ void k_make(uint64_t* recs, uint32_t* keys, uint64_t n, uint64_t base) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t k = fmix32((uint32_t)(base + i) ^ 0x9E3779B9u);
        if (recs) recs[i] = ((base + i) << 32) | k;
        if (keys) keys[i] = k;
    }
}

template <bool MATCH>
__global__ void __launch_bounds__(256) k_part(const uint64_t* __restrict__ recs, uint64_t n, uint64_t* tab,
                                              uint64_t mask, uint8_t* flag, unsigned long long* over) {
    const int lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * 256;
    for (uint64_t t0 = (uint64_t)blockIdx.x * 256 + (threadIdx.x & ~31u); t0 < n; t0 += stride) {
        const uint64_t t = t0 + lane;
        const bool active = t < n;
        const uint64_t w = active ? recs[t] : EMPTY;
        const uint32_t k = (uint32_t)w, op = (uint32_t)(w >> 32);
        uint32_t mx = op;
        if (MATCH) {
            const uint32_t grp = __match_any_sync(FULL, k);
            if (!active) continue;
            if (__popc(grp) > 1) { flag[op] = 1; mx = __reduce_max_sync(grp, op); }
        } else if (!active) continue;
        if (op != mx) continue;
        const uint64_t word = ((uint64_t)k << 32) | op;
        const uint32_t hk = fmix32(k ^ 0x2545F491u);
        uint64_t h = hk & mask;
        uint64_t probe = 0;
        for (; probe <= mask; ++probe) {
            const uint64_t prev = atomicCAS((unsigned long long*)&tab[h], EMPTY, word);
            if (prev == EMPTY) break;
            if ((uint32_t)(prev >> 32) == k) {
                flag[op] = 1; flag[(uint32_t)prev] = 1;
                if (word > prev) atomicMax((unsigned long long*)&tab[h], (unsigned long long)word);
                break;
            }
            h = (h + 1) & mask;
        }
        if (probe > mask) atomicAdd(over, 1ull);
    }
}

// seen / dup bitmaps (B bits each, B a power of two)
__global__ void __launch_bounds__(256) k_seen(const uint32_t* __restrict__ keys, uint64_t n, uint32_t* seen,
                                              uint32_t* dup, uint32_t bmask) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = fmix32(keys[i] ^ 0x2545F491u) & bmask;
        const uint32_t bit = 1u << (p & 31);
        const uint32_t old = atomicOr(&seen[p >> 5], bit);
        if (old & bit) atomicOr(&dup[p >> 5], bit);       // result unused: RED
    }
}
__global__ void __launch_bounds__(256) k_flagged(const uint32_t* __restrict__ keys, uint64_t n,
                                                 const uint32_t* __restrict__ dup, uint32_t bmask,
                                                 unsigned long long* cnt) {
    unsigned c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = fmix32(keys[i] ^ 0x2545F491u) & bmask;
        c += (dup[p >> 5] >> (p & 31)) & 1u;
    }
    c = __reduce_add_sync(FULL, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, (unsigned long long)c);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t N = 1ull << 26, NP = 1ull << 21;
    uint64_t *recs, *tab; uint32_t* keys; uint8_t* flag; unsigned long long* cnt;
    uint32_t *seen, *dup;
    cudaMalloc(&recs, NP * 8); cudaMalloc(&tab, 64ull << 20); cudaMalloc(&keys, N * 4);
    cudaMalloc(&flag, N); cudaMalloc(&cnt, 8 * 4);
    cudaMalloc(&seen, 1ull << 27); cudaMalloc(&dup, 1ull << 27);
    cudaMemset(flag, 0, N);
    k_make<<<sms * 8, 256>>>(recs, nullptr, NP, 0);
    k_make<<<sms * 8, 256>>>(nullptr, keys, N, 0);
    uint8_t* junk; cudaMalloc(&junk, 512ull << 20);       // evicts L2 between trials
    cudaEvent_t e[4];
    for (auto& x : e) cudaEventCreate(&x);
    auto ms = [&](int a, int b) { float t; cudaEventElapsedTime(&t, e[a], e[b]); return t * 1e3f; };
    for (int grid_mul : {4, 8, 16}) {
        for (int variant = 0; variant < 3; ++variant) {
            for (uint64_t tb : {64ull << 20, 32ull << 20}) {   // 16 MiB = 2^21 slots: full at 2^21 ops
                const uint64_t mask = tb / 8 - 1;
                float best_m = 1e9, best_k = 1e9, best_k2 = 1e9;
                for (int rep = 0; rep < 5; ++rep) {
                    cudaMemset(junk, rep, 512ull << 20);
                    cudaEventRecord(e[0]);
                    cudaMemsetAsync(tab, 0xFF, tb);
                    cudaEventRecord(e[1]);
                    if (variant == 1) k_part<false><<<sms * grid_mul, 256>>>(recs, NP, tab, mask, flag, cnt);
                    else k_part<true><<<sms * grid_mul, 256>>>(recs, NP, tab, mask, flag, cnt);
                    cudaEventRecord(e[2]);
                    if (variant == 2) k_part<true><<<sms * grid_mul, 256>>>(recs, NP, tab, mask, flag, cnt);
                    cudaEventRecord(e[3]);
                    cudaEventSynchronize(e[3]);
                    best_m = fminf(best_m, ms(0, 1)); best_k = fminf(best_k, ms(1, 2));
                    best_k2 = fminf(best_k2, ms(2, 3));
                }
                const char* nm[] = {"match", "nomatch", "match,2nd pass"};
                printf("E%d grid %2dx table %2llu MiB: memset %6.1f us  kernel %6.1f us (%5.1f G/s)%s", variant + 1,
                       grid_mul, (unsigned long long)(tb >> 20), best_m, best_k, NP / (best_k * 1e-6) / 1e9, nm[variant]);
                if (variant == 2) printf("  2nd pass (same table, entries present) %6.1f us", best_k2);
                printf("\n");
            }
        }
    }
    for (uint64_t bits : {1ull << 28, 1ull << 29, 1ull << 30}) {
        const uint32_t bmask = (uint32_t)(bits - 1);
        float best[3] = {1e9, 1e9, 1e9};
        unsigned long long hc = 0;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemset(junk, rep, 512ull << 20);
            cudaMemset(cnt, 0, 8);
            cudaEventRecord(e[0]);
            cudaMemsetAsync(seen, 0, bits / 8);
            cudaMemsetAsync(dup, 0, bits / 8);
            cudaEventRecord(e[1]);
            k_seen<<<sms * 8, 256>>>(keys, N, seen, dup, bmask);
            cudaEventRecord(e[2]);
            k_flagged<<<sms * 8, 256>>>(keys, N, dup, bmask, cnt);
            cudaEventRecord(e[3]);
            cudaEventSynchronize(e[3]);
            best[0] = fminf(best[0], ms(0, 1)); best[1] = fminf(best[1], ms(1, 2)); best[2] = fminf(best[2], ms(2, 3));
            cudaMemcpy(&hc, cnt, 8, cudaMemcpyDeviceToHost);
        }
        printf("E4 bitmap %4llu Mbit: clears %6.1f us  seen pass %6.1f us (%5.1f G/s)  flag read %6.1f us  flagged %.4f\n",
               (unsigned long long)(bits >> 20), best[0], best[1], N / (best[1] * 1e-6) / 1e9, best[2], (double)hc / N);
    }
    cudaError_t err = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(err));
    return 0;
}
