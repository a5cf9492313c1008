// Microbenchmark (tuning aid): global RED.ADD throughput into an L2-resident table,
// with the access pattern of "count next digit per output tile" (runs of ~16
// consecutive rows share an output tile; digits random).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

__global__ void k_red(uint32_t* table, uint32_t ntiles, uint64_t n, int mode) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t h = hash32((uint32_t)i);
        uint32_t tile = mode == 0 ? (uint32_t)((i / 16) * 2654435761u % ntiles)   // runs of 16 rows, scattered tiles
                                  : (uint32_t)(i / 4096) % ntiles;                   // sequential tiles
        const uint32_t d = h & 255u;
        atomicAdd(table + (size_t)tile * 256 + d, 1u);
    }
}

__global__ void k_copy(const uint4* a, uint4* b, uint64_t n4) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) b[i] = a[i];
}

int main() {
    const uint64_t n = 157500000ull;
    const uint32_t ntiles = (uint32_t)((n + 4095) / 4096);
    uint32_t* table; cudaMalloc(&table, (size_t)ntiles * 256 * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(table, 0, (size_t)ntiles * 256 * 4);
            cudaEventRecord(a);
            k_red<<<148 * 8, 256>>>(table, ntiles, n, mode);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("RED mode %d: %llu reds in %.3f ms = %.1f G/s (table %.1f MB)\n", mode,
                            (unsigned long long)n, ms, n / ms / 1e6, ntiles * 256 * 4 / 1e6);
        }
    }
    // reference: copy bandwidth
    const uint64_t bytes = 2520000000ull;
    uint4 *x, *y; cudaMalloc(&x, bytes); cudaMalloc(&y, bytes);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        k_copy<<<148 * 8, 256>>>(x, y, bytes / 16);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep == 2) printf("copy %.2f GB: %.3f ms = %.0f GB/s (r+w)\n", bytes / 1e9, ms, 2.0 * bytes / ms / 1e6);
    }
    return 0;
}
