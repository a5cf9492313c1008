// rmx_steps.cuh -- small device steps of the multi-GPU path:
//   k_gather      out[i] = table[idx[i]]         (the K4 remap with a caller table)
//   k_lower_bound first row >= query, rows in the reference's bitwise order
#pragma once

#include "rmx_base.cuh"

namespace rmx {

__global__ void __launch_bounds__(kBlock) k_gather(const uint32_t* table, uint64_t n_table, const uint32_t* idx,
                                                   uint64_t n, uint32_t* out, uint32_t* status) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    bool bad = false;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x; i < n; i += stride) {
        const uint32_t j = __ldcs(idx + i);
        if (j < n_table) out[i] = __ldg(table + j);
        else bad = true;
    }
    if (__any_sync(kFull, bad) && (threadIdx.x & 31u) == 0u) atomicOr(status, RMX_STATUS_INDEX_OUT_OF_RANGE);
}

// Lexicographic compare of D-word rows, component 0 most significant, raw
// unsigned words (primitives.py:23-27).
__device__ __forceinline__ int row_cmp(const uint32_t* a, const uint32_t* b, int D) {
    for (int c = 0; c < D; ++c) {
        if (a[c] != b[c]) return a[c] < b[c] ? -1 : 1;
    }
    return 0;
}

// One thread per query: first position in rows[0..n) (sorted) whose row >= query.
__global__ void k_lower_bound(const uint32_t* rows, uint64_t n, int D, const uint32_t* queries, uint64_t nq,
                              unsigned long long* out) {
    const uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const uint32_t* key = queries + q * D;
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (row_cmp(rows + mid * D, key, D) < 0) lo = mid + 1;
        else hi = mid;
    }
    out[q] = lo;
}

// merge (reference ops.py:29-34): a piece's indices shifted by the vertex
// count of the pieces before it, written into the concatenated index array.
__global__ void __launch_bounds__(kBlock) k_offset_indices(const uint32_t* __restrict__ idx, uint64_t n,
                                                           uint32_t offset, uint32_t* __restrict__ out, int vec) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    uint64_t done = 0;
    if (vec) {
        const uint64_t n4 = n >> 2;
        const uint4* i4 = reinterpret_cast<const uint4*>(idx);
        uint4* o4 = reinterpret_cast<uint4*>(out);
        for (uint64_t i = t0; i < n4; i += stride) {
            const uint4 v = __ldcs(i4 + i);
            __stcs(o4 + i, make_uint4(v.x + offset, v.y + offset, v.z + offset, v.w + offset));
        }
        done = n4 << 2;
    }
    for (uint64_t i = done + t0; i < n; i += stride) out[i] = idx[i] + offset;
}

// Distributed exchange over peer memory (dist.SymmComm): rows [bounds[g],
// bounds[g+1]) of the sorted local array go straight into peer g's symmetric
// receive buffer at row dst_off[g] -- the partition and the NVLink transfer in
// one kernel, no send staging, no NCCL kernel.  One thread per output word:
// reads are coalesced, and so are the stores inside each destination range.
__global__ void __launch_bounds__(kBlock) k_scatter_rows(const uint32_t* __restrict__ src, uint64_t n, uint32_t words,
                                                         const uint64_t* __restrict__ bounds, uint32_t G,
                                                         const uint64_t* __restrict__ dst_ptrs,
                                                         const uint64_t* __restrict__ dst_off) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const uint64_t total = n * words;
    for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x; t < total; t += stride) {
        const uint64_t row = t / words;
        const uint32_t w = static_cast<uint32_t>(t - row * words);
        uint32_t lo = 0, hi = G;  // last g with bounds[g] <= row
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (bounds[mid] <= row) lo = mid;
            else hi = mid;
        }
        uint32_t* dst = reinterpret_cast<uint32_t*>(dst_ptrs[lo]);
        dst[(dst_off[lo] + row - bounds[lo]) * words + w] = src[t];
    }
}

// subset (reference ops.py:59-68) on the device: the selected elements
// (keep[e] != 0) in order.  Reduce-then-scan over tiles of 2048 elements:
// k_keep_count counts per tile, k_rows_scan (rmx_merge.cuh) scans the counts,
// k_keep_compact writes each kept element to its rank.
constexpr uint32_t kKeepTile = 2048;

__global__ void __launch_bounds__(kBlock) k_keep_count(const uint8_t* __restrict__ keep, uint64_t n,
                                                       uint32_t* __restrict__ counts) {
    __shared__ uint32_t s_red[kWarps];
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kKeepTile;
    uint32_t c = 0;
    for (uint64_t e = t0 + threadIdx.x; e < min(n, t0 + kKeepTile); e += kBlock) c += keep[e] ? 1u : 0u;
    c = warp_sum(c);
    if ((threadIdx.x & 31u) == 0u) s_red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kWarps; ++w) t += s_red[w];
        counts[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kBlock) k_keep_compact(const uint32_t* __restrict__ idx, uint64_t n, uint32_t K,
                                                         const uint8_t* __restrict__ keep,
                                                         const uint32_t* __restrict__ prefix,
                                                         uint32_t* __restrict__ out) {
    __shared__ uint32_t s_warp[kWarps];
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kKeepTile;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t running = prefix[blockIdx.x];
    for (uint64_t e0 = t0; e0 < min(n, t0 + kKeepTile); e0 += kBlock) {
        const uint64_t e = e0 + threadIdx.x;
        const bool k = e < n && keep[e];
        const uint32_t bal = __ballot_sync(kFull, k);
        if (lane == 0) s_warp[warp] = __popc(bal);
        __syncthreads();
        uint32_t before = 0, all = 0;
        for (int w = 0; w < kWarps; ++w) {
            before += (static_cast<uint32_t>(w) < warp) ? s_warp[w] : 0u;
            all += s_warp[w];
        }
        __syncthreads();
        if (k) {
            const uint64_t dst = running + before + __popc(bal & lanemask_lt());
            for (uint32_t s = 0; s < K; ++s) out[dst * K + s] = idx[e * K + s];
        }
        running += all;
    }
}

}  // namespace rmx
