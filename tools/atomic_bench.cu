// Micro-benchmark: global atomic throughput on B200 for the owner-election
// design.  2^26 ops on random slots of a table of T words:
// CAS64 (with return), atomicMax64 with return, RED.MAX64 / RED.ADD32 (no
// return), and a plain 8-byte gather for reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/atomic_bench tools/atomic_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t h) {
    h ^= h >> 16; h *= 0x85ebca6bu; h ^= h >> 13; h *= 0xc2b2ae35u; h ^= h >> 16; return h;
}

template <int MODE>
__global__ void k(unsigned long long* tab, uint64_t mask, uint64_t n, unsigned long long* sink) {
    unsigned long long acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t h = mix((uint32_t)i ^ 0x9E3779B9u);
        const uint64_t s = ((uint64_t)h * 2654435761ull) & mask;
        const unsigned long long w = ((unsigned long long)h << 32) | (uint32_t)i;
        if (MODE == 0) acc += atomicCAS(&tab[s], ~0ull, w);
        else if (MODE == 1) acc += atomicMax(&tab[s], w);
        else if (MODE == 2) atomicMax(&tab[s], w);
        else if (MODE == 3) atomicAdd((unsigned int*)&tab[s], 1u);
        else if (MODE == 4) acc += __ldcg(&tab[s]);
        else if (MODE == 5) acc += atomicCAS((unsigned int*)&tab[s], ~0u, (unsigned)i);
    }
    if (acc == 0x12345) *sink = acc;
}

int main() {
    const uint64_t n = 1ull << 26;
    const char* names[] = {"CAS64 ret", "MAX64 ret", "RED.MAX64", "RED.ADD32", "gather64", "CAS32 ret"};
    unsigned long long *tab, *sink;
    cudaMalloc(&tab, 1ull << 30);
    cudaMalloc(&sink, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (uint64_t tb : {8ull << 20, 32ull << 20, 64ull << 20, 1ull << 30}) {
        const uint64_t mask = tb / 8 - 1;
        for (int mode = 0; mode < 6; ++mode) {
            for (int grid_mul : {8, 32}) {
                float best = 1e9;
                for (int rep = 0; rep < 4; ++rep) {
                    cudaMemset(tab, 0xFF, tb);
                    cudaEventRecord(a);
                    switch (mode) {
                        case 0: k<0><<<sms * grid_mul, 256>>>(tab, mask, n, sink); break;
                        case 1: k<1><<<sms * grid_mul, 256>>>(tab, mask, n, sink); break;
                        case 2: k<2><<<sms * grid_mul, 256>>>(tab, mask, n, sink); break;
                        case 3: k<3><<<sms * grid_mul, 256>>>(tab, mask, n, sink); break;
                        case 4: k<4><<<sms * grid_mul, 256>>>(tab, mask, n, sink); break;
                        case 5: k<5><<<sms * grid_mul, 256>>>(tab, mask, n, sink); break;
                    }
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms; cudaEventElapsedTime(&ms, a, b);
                    if (ms < best) best = ms;
                }
                printf("table %5llu MiB  %-10s grid %2dx: %7.3f ms  %6.1f G ops/s\n", (unsigned long long)(tb >> 20),
                       names[mode], grid_mul, best, n / (best * 1e-3) / 1e9);
            }
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
