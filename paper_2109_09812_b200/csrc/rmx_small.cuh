// rmx_small.cuh -- the whole re-index of a small mesh in one CTA.
//
// For V <= kSmallV vertices (D <= kSmallD words each, V * D <= kSmallWords,
// I <= kSmallI index slots) the ~50 launches of the large-mesh pipeline cost
// far more than the work.  One 1024-thread CTA runs every step in shared memory with the same
// semantics (pipeline.py:133-157):
//   mark (pipeline.py:41-51) -> replace unused rows (54-63) -> stable
//   lexicographic sort of (key words, row) by a bitonic network on row ids
//   with the row id as the final tie-break (primitives.py:23-40) -> head
//   flags + scan (72-94) -> unique rows out (97-100) -> map (103-113) ->
//   remap (116-130), plus every ReindexScratch field.
#pragma once

#include "rmx_base.cuh"

namespace rmx {

constexpr int kSmallThreads = 1024;
constexpr uint32_t kSmallV = 8192;            // bitonic network of <= 8192 row ids (<= 4 pairs per thread per step)
constexpr uint32_t kSmallD = 8;
constexpr uint32_t kSmallWords = 24576;       // V * D key words in shared memory (96 KB)
constexpr uint64_t kSmallI = 1ull << 18;
constexpr int kSmallSlots = kSmallV / kSmallThreads;  // sorted slots per thread in the head scan

__host__ __device__ inline size_t small_smem_bytes(uint32_t V, uint32_t D) {
    // keys, sorted ids (u16), map (u32), flags (u8), scan scratch
    return static_cast<size_t>(V) * D * 4 + kSmallV * 2 + static_cast<size_t>(V) * 4 + kSmallV + 64 * 4;
}

struct SmallArgs {
    const uint32_t* vtx;
    uint32_t V;
    uint32_t D;
    const uint32_t* idx;
    uint64_t I;
    uint32_t* out_vtx;
    uint32_t* out_idx;
    unsigned long long* count;
    uint32_t* status;
    rmx_scratch sc;
};

// row a before row b: lexicographic on the cleaned key words, then row id
__device__ __forceinline__ bool small_less(const uint32_t* keys, uint32_t D, uint32_t V, uint32_t a, uint32_t b) {
    if (a >= V) return false;  // padding sorts last
    if (b >= V) return true;
    const uint32_t* ka = keys + a * D;
    const uint32_t* kb = keys + b * D;
    for (uint32_t c = 0; c < D; ++c)
        if (ka[c] != kb[c]) return ka[c] < kb[c];
    return a < b;
}

__global__ void __launch_bounds__(kSmallThreads) k_small(SmallArgs a) {
    uint32_t* smem = dyn_smem<uint32_t>();
    const uint32_t V = a.V, D = a.D;
    uint32_t* s_key = smem;                                       // [V * D]
    uint16_t* s_ord = reinterpret_cast<uint16_t*>(s_key + V * D); // [kSmallV] sorted position -> row
    uint32_t* s_map = reinterpret_cast<uint32_t*>(s_ord + kSmallV); // [V] row -> new index
    uint8_t* s_flag = reinterpret_cast<uint8_t*>(s_map + V);      // [kSmallV] used / head flags
    uint32_t* s_warp = reinterpret_cast<uint32_t*>(s_flag + kSmallV);  // [32] + bad flag
    const uint32_t tid = threadIdx.x;

    for (uint32_t i = tid; i < kSmallV; i += kSmallThreads) s_flag[i] = 0;
    if (tid == 0) s_warp[32] = 0u;
    __syncthreads();
    // ---- mark
    bool bad = false;
    for (uint64_t k = tid; k < a.I; k += kSmallThreads) {
        const uint32_t x = a.idx[k];
        if (x < V) s_flag[x] = 1;
        else bad = true;
    }
    if (bad) atomicOr(s_warp + 32, 1u);
    __syncthreads();
    if (s_warp[32]) {
        if (tid == 0) atomicOr(a.status, RMX_STATUS_INDEX_OUT_OF_RANGE);
        return;
    }
    if (a.sc.is_used)
        for (uint32_t i = tid; i < V; i += kSmallThreads) a.sc.is_used[i] = s_flag[i];
    // ---- cleaned keys: unused rows take the replacement row vertices[elements[0,0]]
    const uint32_t r0 = a.idx[0];
    for (uint32_t w = tid; w < V * D; w += kSmallThreads) {
        const uint32_t i = w / D, c = w - i * D;
        s_key[w] = s_flag[i] ? a.vtx[w] : a.vtx[r0 * D + c];
    }
    for (uint32_t i = tid; i < kSmallV; i += kSmallThreads) s_ord[i] = static_cast<uint16_t>(i);
    __syncthreads();
    // ---- bitonic sort of row ids (N = next power of two >= V; ids >= V are padding)
    uint32_t N = 1;
    while (N < V) N <<= 1;
    for (uint32_t k = 2; k <= N; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t t = tid; t < N / 2; t += kSmallThreads) {
                const uint32_t lo = 2 * j * (t / j) + (t % j), hi = lo + j;
                const bool up = (lo & k) == 0;
                const uint32_t x = s_ord[lo], y = s_ord[hi];
                if (small_less(s_key, D, V, y, x) == up) {
                    s_ord[lo] = static_cast<uint16_t>(y);
                    s_ord[hi] = static_cast<uint16_t>(x);
                }
            }
            __syncthreads();
        }
    }
    // ---- head flags and their inclusive scan -> new index per slot
    uint32_t local[kSmallSlots];
    uint32_t sum = 0;
#pragma unroll
    for (int r = 0; r < kSmallSlots; ++r) {
        const uint32_t p = kSmallSlots * tid + r;
        uint32_t h = 0;
        if (p < V) {
            if (p == 0) {
                h = 1;
            } else {
                const uint32_t* ka = s_key + s_ord[p] * D;
                const uint32_t* kb = s_key + s_ord[p - 1] * D;
                for (uint32_t c = 0; c < D; ++c)
                    if (ka[c] != kb[c]) {
                        h = 1;
                        break;
                    }
            }
        }
        local[r] = h;
        sum += h;
    }
    uint32_t total;
    const uint32_t excl = block_exclusive_scan<kSmallThreads / 32>(sum, s_warp, total);
    __syncthreads();
    uint32_t run = excl;
#pragma unroll
    for (int r = 0; r < kSmallSlots; ++r) {
        const uint32_t p = kSmallSlots * tid + r;
        run += local[r];
        if (p < V) {
            const uint32_t row = s_ord[p];
            const uint32_t nidx = run - 1u;
            s_map[row] = nidx;
            if (local[r])
                for (uint32_t c = 0; c < D; ++c) a.out_vtx[nidx * D + c] = s_key[row * D + c];
            if (a.sc.org_id) a.sc.org_id[p] = row;
            if (a.sc.nodup) a.sc.nodup[p] = static_cast<uint8_t>(local[r]);
            if (a.sc.new_idx) a.sc.new_idx[p] = nidx;
            if (a.sc.perm) a.sc.perm[row] = p;
        }
    }
    if (tid == 0) *a.count = total;
    __syncthreads();
    // ---- remap
    for (uint64_t k = tid; k < a.I; k += kSmallThreads) a.out_idx[k] = s_map[a.idx[k]];
}

}  // namespace rmx
