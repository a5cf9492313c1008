// Microbenchmarks (tuning aid, not product): warp-level stable ranking options for 8-bit digits.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t lanemask_lt() { uint32_t m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }

// digits are precomputed in a register array (no hash in the loop)
template <int MODE, int DISTINCT>
__global__ void k_rank(uint32_t* out, int iters) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t dg[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) dg[j] = ((lane * 2654435761u + j * 40503u + blockIdx.x) >> 7) % DISTINCT;
    uint32_t acc = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint32_t d = (dg[j] + i) & 255;
            uint32_t peers;
            if (MODE == 0) {
                peers = __match_any_sync(0xffffffffu, d);
            } else if (MODE == 1) {
                peers = 0xffffffffu;
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1);
                    peers &= ((d >> b) & 1) ? bb : ~bb;
                }
            } else if (MODE == 2) {
                // uniform fast path, else ballots
                const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
                if (__all_sync(0xffffffffu, d == d0)) peers = 0xffffffffu;
                else {
                    peers = 0xffffffffu;
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1);
                        peers &= ((d >> b) & 1) ? bb : ~bb;
                    }
                }
            } else if (MODE == 4) {
                // ballots via redux.sync OR of lane bits
                peers = 0xffffffffu;
                const uint32_t lb = 1u << lane;
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    const uint32_t bb = __reduce_or_sync(0xffffffffu, ((d >> b) & 1) ? lb : 0u);
                    peers &= ((d >> b) & 1) ? bb : ~bb;
                }
            } else if (MODE == 5) {
                // half ballots, half redux (two different units)
                peers = 0xffffffffu;
                const uint32_t lb = 1u << lane;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1);
                    peers &= ((d >> b) & 1) ? bb : ~bb;
                }
#pragma unroll
                for (int b = 4; b < 8; ++b) {
                    const uint32_t bb = __reduce_or_sync(0xffffffffu, ((d >> b) & 1) ? lb : 0u);
                    peers &= ((d >> b) & 1) ? bb : ~bb;
                }
            } else if (MODE == 6) {
                // nibble matches: peers = match(low nibble) & match(high nibble)... (exact: match on d>>4 and d&15)
                peers = __match_any_sync(0xffffffffu, d & 15u) & __match_any_sync(0xffffffffu, d >> 4);
            } else {
                // bitonic sort of (d<<5|lane) across the warp, then peers from neighbours
                uint32_t k = (d << 5) | lane;
#pragma unroll
                for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
                    for (int stride = size >> 1; stride > 0; stride >>= 1) {
                        const uint32_t o = __shfl_xor_sync(0xffffffffu, k, stride);
                        const bool up = ((lane & size) == 0);
                        const bool lower = (lane & stride) == 0;
                        const uint32_t mn = min(k, o), mx = max(k, o);
                        k = (lower == up) ? mn : mx;
                    }
                }
                peers = k;  // stand-in: sorted key; a real rank needs a scatter back (1 more shfl)
            }
            acc += __popc(peers & lanemask_lt()) + peers;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <typename K>
void run(const char* name, K kern) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out; cudaMalloc(&out, 1 << 26);
    const int iters = 256, bps = 4, threads = 256;
    const int grid = sms * bps;
    kern<<<grid, threads>>>(out, iters);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<grid, threads>>>(out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double warp_rounds = double(grid) * threads / 32 * iters * 16;
    double cyc = ms * 1e-3 * 1965e6;
    printf("%-34s %8.3f ms  %6.1f SM-cycles per warp-round  (%.2f rows/cycle/SM)\n", name, ms,
           cyc * sms / warp_rounds, warp_rounds * 32 / cyc / sms);
    cudaFree(out);
}

__global__ void k_atom_order(uint32_t* out) {
    __shared__ uint32_t h[4];
    if (threadIdx.x < 4) h[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    uint32_t bad = 0;
    for (int i = 0; i < 1000; ++i) {
        const uint32_t d = (lane * 7 + i) & 3;
        const uint32_t old = atomicAdd(&h[d], 1);
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t lead = __ffs(peers) - 1;
        const uint32_t base = __shfl_sync(0xffffffffu, old, lead);
        bad += (old - base) != __popc(peers & lanemask_lt());
        __syncwarp();
    }
    atomicAdd(out, bad);
}

int main() {
    run("match 256 distinct", k_rank<0, 256>);
    run("match 32 distinct", k_rank<0, 32>);
    run("match 8 distinct", k_rank<0, 8>);
    run("match 1 distinct", k_rank<0, 1>);
    run("ballot8 256", k_rank<1, 256>);
    run("ballot8 8", k_rank<1, 8>);
    run("uniform+ballot8 256", k_rank<2, 256>);
    run("uniform+ballot8 1", k_rank<2, 1>);
    run("bitonic32 256", k_rank<3, 256>);
    run("redux8 256", k_rank<4, 256>);
    run("ballot4+redux4 256", k_rank<5, 256>);
    run("match nibbles 256", k_rank<6, 256>);
    uint32_t* o; cudaMalloc(&o, 4); cudaMemset(o, 0, 4);
    k_atom_order<<<148, 256>>>(o);
    uint32_t bad; cudaMemcpy(&bad, o, 4, cudaMemcpyDeviceToHost);
    printf("same-address smem atomics out of lane order: %u of %u\n", bad, 148 * 256 * 1000);
    return 0;
}
