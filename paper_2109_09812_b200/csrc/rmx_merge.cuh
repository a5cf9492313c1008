// rmx_merge.cuh -- sorted-run merge + unique for the multi-GPU exchange.
//
// After the all-to-all of dist.py step 3 a rank holds G runs of rows, each run
// sorted and duplicate-free (one sender's local unique keys of this rank's
// key range).  Step 4 needs the sorted unique keys of all of them and the rank
// of every received row.  Instead of re-sorting (the full LSD pipeline), the
// runs are merged pairwise with a merge path (log2 G rounds, each a read and
// a write of the rows) and duplicates -- the same key from several senders,
// adjacent after the merge -- are collapsed in one compaction:
//
//   k_merge_path     one CTA per 2048 output rows: diagonal split of (A, B)
//                    by binary search, the two slices staged in shared memory,
//                    a per-thread split inside the block, rows written out.
//                    Rows are W words: D key words (component 0 most
//                    significant) + the arrival position.  Ties take A first.
//   k_rows_heads     per 2048-row tile: number of rows whose key differs from
//                    the previous row's
//   k_rows_scan      exclusive scan of the tile counts (one CTA), total
//   k_rows_unique    unique keys out, rank of every arrival position
#pragma once

#include "rmx_base.cuh"

namespace rmx {

constexpr uint32_t kMergeTile = 2048;  // output rows per CTA (merge and unique)
constexpr uint32_t kMergeMaxW = 9;     // D <= 8 key words + arrival position

// key(a) < key(b) on the first D words
__device__ __forceinline__ bool rows_less(const uint32_t* a, const uint32_t* b, uint32_t D) {
    for (uint32_t c = 0; c < D; ++c)
        if (a[c] != b[c]) return a[c] < b[c];
    return false;
}

// number of A rows among the first `diag` merged rows (A before B on ties)
__device__ __forceinline__ uint64_t merge_split(const uint32_t* A, uint64_t na, const uint32_t* B, uint64_t nb,
                                                uint32_t W, uint32_t D, uint64_t diag) {
    uint64_t lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
    while (lo < hi) {
        const uint64_t i = (lo + hi) >> 1;  // candidate: i rows of A, diag - i of B
        // take more A while A[i] <= B[diag - i - 1]  (ties to A)
        if (!rows_less(B + (diag - i - 1) * W, A + i * W, D)) lo = i + 1;
        else hi = i;
    }
    return lo;
}

// rows of D key words + arrival position, from the keys of the runs (one row per thread)
template <int W>
__global__ void __launch_bounds__(kBlock) k_merge_rows_init(const uint32_t* __restrict__ keys, uint64_t n,
                                                             uint32_t org0, uint32_t* __restrict__ rows) {
    constexpr int D = W - 1;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    for (uint64_t r = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x; r < n; r += stride) {
        uint32_t* dst = rows + r * W;
#pragma unroll
        for (int c = 0; c < D; ++c) dst[c] = __ldcs(keys + r * D + c);
        dst[D] = org0 + static_cast<uint32_t>(r);
    }
}

// merge-path split at every CTA boundary (rows of stride S words; one thread each: the ~log2(n) dependent
// global loads run in parallel here instead of at the head of every merge CTA)
__global__ void __launch_bounds__(kBlock) k_merge_splits(const uint32_t* __restrict__ A, uint64_t na,
                                                          const uint32_t* __restrict__ B, uint64_t nb, uint32_t W,
                                                          uint32_t D, uint64_t* __restrict__ splits, uint32_t nsplits) {
    const uint32_t t = blockIdx.x * kBlock + threadIdx.x;
    if (t < nsplits) splits[t] = merge_split(A, na, B, nb, W, D, min(na + nb, static_cast<uint64_t>(t) * kMergeTile));
}

// Shared-memory row r lives at padded(r) * W ... with one pad word per 8 rows, so
// that threads walking rows 8 apart (one merge stretch each) hit distinct banks.
__device__ __forceinline__ uint32_t pad_row(uint32_t r, uint32_t W) { return r * W + (r >> 3); }

// key(row a) < key(row b) for padded shared-memory rows
__device__ __forceinline__ bool srows_less(const uint32_t* s, uint32_t a, uint32_t b, uint32_t W, uint32_t D) {
    const uint32_t* ka = s + pad_row(a, W);
    const uint32_t* kb = s + pad_row(b, W);
    for (uint32_t c = 0; c < D; ++c)
        if (ka[c] != kb[c]) return ka[c] < kb[c];
    return false;
}

// FROM_KEYS (first round): A and B are runs of the received keys (D words per row, row ids
// a_org / b_org onwards); the arrival position becomes the W-th word as the rows are staged.
template <int W, bool FROM_KEYS>
__global__ void __launch_bounds__(kBlock) k_merge_path(const uint32_t* __restrict__ A, uint64_t na,
                                                        const uint32_t* __restrict__ B, uint64_t nb,
                                                        uint32_t a_org, uint32_t b_org,
                                                        const uint64_t* __restrict__ splits,
                                                        uint32_t* __restrict__ out) {
    constexpr uint32_t D = W - 1;
    constexpr uint32_t S = FROM_KEYS ? D : W;  // input row stride
    // input rows (A slice then B slice), then the merged rows, both padded
    uint32_t* s_rows = dyn_smem<uint32_t>();
    const uint32_t span = pad_row(kMergeTile, W) + 1;
    uint32_t* s_out = s_rows + span;
    const uint64_t n = na + nb;
    const uint64_t d0 = static_cast<uint64_t>(blockIdx.x) * kMergeTile;
    const uint64_t d1 = min(n, d0 + kMergeTile);
    const uint64_t a0 = splits[blockIdx.x], a1 = splits[blockIdx.x + 1];
    const uint64_t b0 = d0 - a0, b1 = d1 - a1;
    const uint32_t la = static_cast<uint32_t>(a1 - a0), lb = static_cast<uint32_t>(b1 - b0);
    const uint32_t total = la + lb;
    for (uint32_t w = threadIdx.x; w < la * S; w += kBlock) {
        const uint32_t r = w / S;
        s_rows[pad_row(r, W) + (w - r * S)] = A[a0 * S + w];
    }
    for (uint32_t w = threadIdx.x; w < lb * S; w += kBlock) {
        const uint32_t r = w / S;
        s_rows[pad_row(la + r, W) + (w - r * S)] = B[b0 * S + w];
    }
    if (FROM_KEYS) {
        for (uint32_t r = threadIdx.x; r < la; r += kBlock) s_rows[pad_row(r, W) + D] = a_org + static_cast<uint32_t>(a0) + r;
        for (uint32_t r = threadIdx.x; r < lb; r += kBlock)
            s_rows[pad_row(la + r, W) + D] = b_org + static_cast<uint32_t>(b0) + r;
    }
    __syncthreads();
    // thread t merges outputs [8t, 8t + 8): one split search, then a sequential merge with the
    // two candidate rows held in registers (one shared-memory row load per output)
    constexpr uint32_t kPer = kMergeTile / kBlock;
    const uint32_t k0 = threadIdx.x * kPer;
    if (k0 < total) {
        uint32_t lo = k0 > lb ? k0 - lb : 0, hi = k0 < la ? k0 : la;  // split at k0 (A first on ties)
        while (lo < hi) {
            const uint32_t i = (lo + hi) >> 1;
            if (!srows_less(s_rows, la + (k0 - i - 1), i, W, D)) lo = i + 1;
            else hi = i;
        }
        uint32_t i = lo, j = k0 - lo;
        uint32_t ra[W], rb[W];
        auto load = [&](uint32_t (&r)[W], uint32_t row) {
            const uint32_t* p = s_rows + pad_row(row, W);
#pragma unroll
            for (int c = 0; c < W; ++c) r[c] = p[c];
        };
        if (i < la) load(ra, i);
        if (j < lb) load(rb, la + j);
        const uint32_t kend = min(k0 + kPer, total);
        for (uint32_t k = k0; k < kend; ++k) {
            bool b_less = false;  // key(rb) < key(ra)
#pragma unroll
            for (int c = static_cast<int>(D) - 1; c >= 0; --c)
                b_less = (rb[c] != ra[c]) ? (rb[c] < ra[c]) : b_less;
            const bool take_a = j >= lb || (i < la && !b_less);
            uint32_t* dp = s_out + pad_row(k, W);
            if (take_a) {
#pragma unroll
                for (int c = 0; c < W; ++c) dp[c] = ra[c];
                if (++i < la) load(ra, i);
            } else {
#pragma unroll
                for (int c = 0; c < W; ++c) dp[c] = rb[c];
                if (++j < lb) load(rb, la + j);
            }
        }
    }
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < total * W; w += kBlock) {  // coalesced write-out
        const uint32_t r = w / W;
        out[d0 * W + w] = s_out[pad_row(r, W) + (w - r * W)];
    }
}

__global__ void __launch_bounds__(kBlock) k_rows_heads(const uint32_t* __restrict__ rows, uint64_t n, uint32_t W,
                                                        uint32_t D, uint32_t* __restrict__ counts) {
    __shared__ uint32_t s_red[kWarps];
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kMergeTile;
    uint32_t cnt = 0;
    for (uint64_t r = t0 + threadIdx.x; r < min(n, t0 + kMergeTile); r += kBlock) {
        bool head = r == 0;
        if (!head) {
            const uint32_t* a = rows + r * W;
            const uint32_t* b = a - W;
            for (uint32_t c = 0; c < D; ++c) head = head || a[c] != b[c];
        }
        cnt += head ? 1u : 0u;
    }
    cnt = warp_sum(cnt);
    if ((threadIdx.x & 31u) == 0u) s_red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (int w = 0; w < kWarps; ++w) tot += s_red[w];
        counts[blockIdx.x] = tot;
    }
}

// exclusive scan of counts[0, ntiles) in place (one CTA of 1024), total -> *total
__global__ void __launch_bounds__(1024) k_rows_scan(uint32_t* counts, uint32_t ntiles, unsigned long long* total) {
    __shared__ uint32_t s_warp[32];
    const uint32_t tot = block_scan_counts(counts, ntiles, s_warp);
    if (threadIdx.x == 0) *total = tot;
}

__global__ void __launch_bounds__(kBlock) k_rows_unique(const uint32_t* __restrict__ rows, uint64_t n, uint32_t W,
                                                         uint32_t D, const uint32_t* __restrict__ prefix,
                                                         uint32_t* __restrict__ out_keys, uint32_t* __restrict__ rank_of) {
    __shared__ uint32_t s_warp[kWarps];
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kMergeTile;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t running = prefix[blockIdx.x];
    for (uint64_t r0 = t0; r0 < min(n, t0 + kMergeTile); r0 += kBlock) {
        const uint64_t r = r0 + threadIdx.x;
        bool head = false;
        if (r < n) {
            head = r == 0;
            if (!head) {
                const uint32_t* a = rows + r * W;
                const uint32_t* b = a - W;
                for (uint32_t c = 0; c < D; ++c) head = head || a[c] != b[c];
            }
        }
        const uint32_t bal = __ballot_sync(kFull, head);
        if (lane == 0) s_warp[warp] = __popc(bal);
        __syncthreads();
        uint32_t before = 0, all = 0;
        for (int w = 0; w < kWarps; ++w) {
            before += (static_cast<uint32_t>(w) < warp) ? s_warp[w] : 0u;
            all += s_warp[w];
        }
        __syncthreads();
        if (r < n) {
            const uint32_t nidx = running + before + __popc(bal & lanemask_le()) - 1u;
            const uint32_t* row = rows + r * W;
            if (head)
                for (uint32_t c = 0; c < D; ++c) out_keys[static_cast<uint64_t>(nidx) * D + c] = row[c];
            rank_of[row[D]] = nidx;
        }
        running += all;
    }
}

}  // namespace rmx
