// Microbenchmark (DESIGN.md §11 "beyond the 256 B probe"): how fast are the
// access patterns a tag-filtered probe would need, on the cfg2 geometry
// (2,207,529 buckets of 256 B = 565 MB; a 32 B tag sector per bucket = 70 MB)?
//   mode 0: one random 256 B bucket per op, 4 lanes x 64 B (today's probe)
//   mode 1: one random 32 B sector of the bucket array per op (a lone slot read)
//   mode 2: the bucket's 32 B tag sector (tag array), then one 32 B sector of
//           the bucket chosen by it (dependent) -- a tag-filtered lookup hit
//   mode 3: tag sector only
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sector_bench tools/sector_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
    h ^= h >> 16; h *= 0x85ebca6bu; h ^= h >> 13; h *= 0xc2b2ae35u; h ^= h >> 16; return h;
}
__device__ __forceinline__ void ld4(const uint64_t* p, uint64_t& a, uint64_t& b, uint64_t& c, uint64_t& d) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}

template <int MODE>
__global__ void __launch_bounds__(256) k_bench(const uint64_t* __restrict__ buckets, const uint64_t* __restrict__ tags,
                                               uint64_t nb, uint64_t n, uint32_t* __restrict__ out) {
    const uint64_t tid = (uint64_t)blockIdx.x * 256 + threadIdx.x;
    const uint64_t nth = (uint64_t)gridDim.x * 256;
    if (MODE == 0) {                       // 4 lanes per op, 64 B each
        const uint64_t grp = tid >> 2, ngrp = nth >> 2;
        const int gl = threadIdx.x & 3;
        for (uint64_t i = grp; i < n; i += ngrp) {
            const uint64_t b = ((uint64_t)fmix32((uint32_t)i) * nb) >> 32;
            uint64_t a0, a1, a2, a3, c0, c1, c2, c3;
            ld4(buckets + b * 32 + gl * 8, a0, a1, a2, a3);
            ld4(buckets + b * 32 + gl * 8 + 4, c0, c1, c2, c3);
            uint32_t x = (uint32_t)(a0 ^ a1 ^ a2 ^ a3 ^ c0 ^ c1 ^ c2 ^ c3);
            x ^= __shfl_xor_sync(0xffffffffu, x, 1);
            x ^= __shfl_xor_sync(0xffffffffu, x, 2);
            if (gl == 0) out[i] = x;
        }
    } else {
        for (uint64_t i = tid; i < n; i += nth) {
            const uint32_t h = fmix32((uint32_t)i);
            const uint64_t b = ((uint64_t)h * nb) >> 32;
            uint32_t x = 0;
            uint32_t slot = (h >> 3) & 31;
            if (MODE == 2 || MODE == 3) {
                uint64_t t0, t1, t2, t3;
                ld4(tags + b * 4, t0, t1, t2, t3);
                x = (uint32_t)(t0 ^ t1 ^ t2 ^ t3);
                slot = (slot ^ x) & 31;
            }
            if (MODE == 1 || MODE == 2) {
                uint64_t w;
                asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(w) : "l"(buckets + b * 32 + slot));
                x ^= (uint32_t)w;
            }
            out[i] = x;
        }
    }
}

int main() {
    const uint64_t nb = 2207529, n = 1ull << 26;
    uint64_t *buckets, *tags;
    uint32_t* out;
    cudaMalloc(&buckets, nb * 256);
    cudaMalloc(&tags, nb * 32);
    cudaMalloc(&out, n * 4);
    cudaMemset(buckets, 1, nb * 256);
    cudaMemset(tags, 2, nb * 32);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[4] = {"256B bucket (4 lanes x 64B)", "one 32B bucket sector", "tag sector -> 32B slot sector",
                            "tag sector only"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int occ = 4; occ <= 8; occ += 4) {
            const int grid = sms * occ;
            float best = 1e9f;
            for (int rep = 0; rep < 6; ++rep) {
                cudaEventRecord(a);
                switch (mode) {
                    case 0: k_bench<0><<<grid, 256>>>(buckets, tags, nb, n, out); break;
                    case 1: k_bench<1><<<grid, 256>>>(buckets, tags, nb, n, out); break;
                    case 2: k_bench<2><<<grid, 256>>>(buckets, tags, nb, n, out); break;
                    default: k_bench<3><<<grid, 256>>>(buckets, tags, nb, n, out); break;
                }
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                if (rep && ms < best) best = ms;
            }
            printf("{\"mode\": %d, \"what\": \"%s\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"G_ops_per_s\": %.2f}\n", mode,
                   names[mode], occ, best, n / (best * 1e-3) / 1e9);
        }
    }
    return 0;
}
