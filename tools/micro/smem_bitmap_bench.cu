// Microbenchmark (tuning aid, not product): the smem-window presence bitmap -- per CTA a 2^20-bit
// (128 KB) bitmap in shared memory, 157.5M random keys split into windows of ~38K keys: zero, mark
// (atomicOr), per-word prefix (u16 within 1024-bit blocks + block prefix), rank every key.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/smem_bitmap_bench tools/micro/smem_bitmap_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}
constexpr int NT = 1024;
constexpr uint32_t WBITS = 20, WWORDS = 1u << (WBITS - 5);

__global__ void k_keys(uint32_t* keys, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        keys[i] = hash32(i * 2654435761u + 7u) & ((1u << WBITS) - 1u);
}

template <int MODE>  // 0: zero+mark only, 1: + prefix + rank
__global__ void __launch_bounds__(NT, 1) k_win(const uint32_t* __restrict__ keys, uint32_t* out, uint32_t n, uint32_t nwin) {
    extern __shared__ uint32_t sm[];
    uint32_t* bm = sm;                                           // WWORDS words
    uint16_t* wpre = reinterpret_cast<uint16_t*>(bm + WWORDS);   // WWORDS u16
    uint32_t* bpre = reinterpret_cast<uint32_t*>(wpre + WWORDS); // WWORDS / 32
    __shared__ uint32_t s_w[32];
    const uint32_t per = n / nwin;
    for (uint32_t w = blockIdx.x; w < nwin; w += gridDim.x) {
        for (uint32_t i = threadIdx.x; i < WWORDS / 4; i += NT) reinterpret_cast<uint4*>(bm)[i] = make_uint4(0, 0, 0, 0);
        __syncthreads();
        const uint32_t r0 = w * per, r1 = r0 + per;
        for (uint32_t i = r0 + threadIdx.x; i < r1; i += NT) {
            const uint32_t k = __ldcs(keys + i);
            atomicOr(bm + (k >> 5), 1u << (k & 31u));
        }
        __syncthreads();
        if (MODE == 1) {
            // thread t: block t of 32 words
            const uint32_t b = threadIdx.x;
            uint32_t run = 0;
            for (int j = 0; j < 32; ++j) {
                wpre[b * 32 + j] = static_cast<uint16_t>(run);
                run += __popc(bm[b * 32 + j]);
            }
            uint32_t x = run;
            for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, x, o); if ((threadIdx.x & 31) >= o) x += y; }
            if ((threadIdx.x & 31) == 31) s_w[threadIdx.x >> 5] = x;
            __syncthreads();
            uint32_t before = 0;
            for (int q = 0; q < 32; ++q) before += q < (int)(threadIdx.x >> 5) ? s_w[q] : 0u;
            bpre[b] = before + x - run;
            __syncthreads();
            for (uint32_t i = r0 + threadIdx.x; i < r1; i += NT) {
                const uint32_t k = __ldcs(keys + i);
                const uint32_t wd = k >> 5;
                out[i] = bpre[wd >> 5] + wpre[wd] + __popc(bm[wd] & ((1u << (k & 31u)) - 1u));
            }
            __syncthreads();
        }
    }
}

int main() {
    const uint32_t n = 157500000u, nwin = 4096;
    uint32_t *keys, *out;
    cudaMalloc(&keys, (size_t)n * 4);
    cudaMalloc(&out, (size_t)n * 4);
    k_keys<<<148 * 8, 256>>>(keys, n);
    const size_t smem = WWORDS * 4 + WWORDS * 2 + WWORDS / 32 * 4;
    cudaFuncSetAttribute(k_win<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_win<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float t0 = 0, t1 = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        k_win<0><<<148, NT, smem>>>(keys, out, n, nwin);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&t0, a, b);
        cudaEventRecord(a);
        k_win<1><<<148, NT, smem>>>(keys, out, n, nwin);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&t1, a, b);
    }
    printf("smem %zu B; zero+mark %.3f ms; zero+mark+prefix+rank %.3f ms; %s\n", smem, t0, t1,
           cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
