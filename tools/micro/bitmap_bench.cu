// Microbenchmark (tuning aid, not product): random atomicOr marks into a presence bitmap and random
// bitmap-word lookups, 157.5M keys, for bitmap sizes from L2-resident to HBM-sized, with keys in
// random order or grouped into 256 consecutive windows (an MSD partition's output order).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/bitmap_bench tools/micro/bitmap_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

__global__ void k_keys(uint32_t* keys, uint32_t n, int bits, int grouped) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t h = hash32(i * 2654435761u + 12345u);
        uint32_t k = bits >= 32 ? h : (h & ((1u << bits) - 1u));
        if (grouped && bits > 8) {  // window w = i / (n / 256) holds the top 8 bits
            const uint32_t w = (uint32_t)((uint64_t)i * 256 / n);
            k = (w << (bits - 8)) | (k & ((1u << (bits - 8)) - 1u));
        }
        keys[i] = k;
    }
}

__global__ void k_mark(const uint32_t* __restrict__ keys, uint32_t* bm, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t k = __ldcs(keys + i);
        atomicOr(bm + (k >> 5), 1u << (k & 31u));
    }
}

__global__ void k_look(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ bm, uint32_t* out, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t k = __ldcs(keys + i);
        const uint32_t w = __ldg(bm + (k >> 5));
        out[i] = __popc(w & ((1u << (k & 31u)) - 1u));
    }
}

int main() {
    const uint32_t n = 157500000u;
    uint32_t *keys, *bm, *out;
    cudaMalloc(&keys, (size_t)n * 4);
    cudaMalloc(&out, (size_t)n * 4);
    cudaMalloc(&bm, (size_t)1 << 29);  // 2^32 bits
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = 148 * 8;
    for (int grouped = 0; grouped < 2; ++grouped) {
        for (int bits : {21, 24, 27, 29, 30, 32}) {
            k_keys<<<grid, 256>>>(keys, n, bits, grouped);
            const size_t bytes = ((size_t)1 << bits) / 8;
            float tm = 0, tl = 0;
            for (int rep = 0; rep < 3; ++rep) {
                cudaMemset(bm, 0, bytes < 4 ? 4 : bytes);
                cudaEventRecord(a);
                k_mark<<<grid, 256>>>(keys, bm, n);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&tm, a, b);
                cudaEventRecord(a);
                k_look<<<grid, 256>>>(keys, bm, out, n);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&tl, a, b);
            }
            printf("%s bits %2d (bitmap %8.1f MB): mark %.3f ms (%.0f G/s), lookup %.3f ms (%.0f G/s)\n",
                   grouped ? "grouped" : "random ", bits, bytes / 1e6, tm, n / tm / 1e6, tl, n / tl / 1e6);
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
