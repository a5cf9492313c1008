// Microbenchmarks (tuning aid, not product): shared-memory atomic throughput by
// address pattern, match.any throughput, ballot multi-split throughput.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

// mode 0: random bin of 256; 1: same bin per warp; 2: 4 distinct bins per warp; 3: 16 distinct
template <int MODE>
__global__ void k_atom(uint32_t* out, int iters) {
    __shared__ uint32_t h[256];
    h[threadIdx.x & 255] = 0;
    __syncthreads();
    uint32_t x = hash32(blockIdx.x * 1024 + threadIdx.x);
    for (int i = 0; i < iters; ++i) {
        x = hash32(x + i);
        uint32_t d;
        if (MODE == 0) d = x & 255;
        else if (MODE == 1) d = (i * 7) & 255;
        else if (MODE == 2) d = ((x & 3) * 37 + i) & 255;
        else d = ((x & 15) * 13 + i) & 255;
        atomicAdd(&h[d], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 256) atomicAdd(out + threadIdx.x, h[threadIdx.x]);
}

template <int MODE>
__global__ void k_match(uint32_t* out, int iters) {
    uint32_t x = hash32(blockIdx.x * 1024 + threadIdx.x), acc = 0;
    for (int i = 0; i < iters; ++i) {
        x = hash32(x + i);
        uint32_t d = MODE == 0 ? (x & 255) : ((x & 3) + i) & 255;
        acc += __match_any_sync(0xffffffffu, d);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// independent matches (ILP 8)
__global__ void k_match8(uint32_t* out, int iters) {
    uint32_t x = hash32(blockIdx.x * 1024 + threadIdx.x), acc = 0;
    for (int i = 0; i < iters; i += 8) {
        uint32_t d[8], m[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) { x = hash32(x + i + j); d[j] = x & 255; }
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = __match_any_sync(0xffffffffu, d[j]);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc += m[j];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_ballot(uint32_t* out, int iters) {
    uint32_t x = hash32(blockIdx.x * 1024 + threadIdx.x), acc = 0;
    for (int i = 0; i < iters; ++i) {
        x = hash32(x + i);
        uint32_t d = x & 255, peers = 0xffffffffu;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1);
            peers &= ((d >> b) & 1) ? bb : ~bb;
        }
        acc += peers;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_base(uint32_t* out, int iters) {
    uint32_t x = hash32(blockIdx.x * 1024 + threadIdx.x), acc = 0;
    for (int i = 0; i < iters; ++i) { x = hash32(x + i); acc += x & 255; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <typename K>
void run(const char* name, K kern, int blocks_per_sm, int threads) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out; cudaMalloc(&out, 1 << 26);
    const int iters = 4096;
    const int grid = sms * blocks_per_sm;
    kern<<<grid, threads>>>(out, iters);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<grid, threads>>>(out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = double(grid) * threads * iters;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double cyc = ms * 1e-3 * 1965e6;
    printf("%-28s %8.3f ms  %7.2f lane-ops/cycle/SM  (%d warps/SM)\n", name, ms, ops / cyc / sms,
           blocks_per_sm * threads / 32);
    cudaFree(out);
}

int main() {
    for (int bps : {2, 4, 8}) {
        run("base(hash only)", k_base, bps, 256);
        run("atom random256", k_atom<0>, bps, 256);
        run("atom same-addr/warp", k_atom<1>, bps, 256);
        run("atom 4 addr/warp", k_atom<2>, bps, 256);
        run("atom 16 addr/warp", k_atom<3>, bps, 256);
        run("match random256", k_match<0>, bps, 256);
        run("match 4 distinct", k_match<1>, bps, 256);
        run("match ILP8", k_match8, bps, 256);
        run("ballot8 multisplit", k_ballot, bps, 256);
    }
    return 0;
}
