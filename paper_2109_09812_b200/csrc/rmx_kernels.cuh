// rmx_kernels.cuh -- the sm_100a kernels of the re-indexing pipeline.
//
//   K1   k_mark         isUsed scatter over the index buffer + range check
//                       (reference mark_used pipeline.py:41-51, require_valid mesh.py:103-105)
//   K1b  k_build_rows   unused -> replacement, AoS (key words, origin) rows,
//                       per-component varying-bit masks, component D-1 digit
//                       histograms (overwrite_unused pipeline.py:54-63,
//                       fill_sequence primitives.py:16-20)
//   plan k_plan         digit-pass skipping, ping-pong schedule, pass chaining
//   hist k_first_hist   histogram of the first executed pass if K1b lacks it
//   K2   k_sort_pass    one onesweep LSD pass: double-buffered TMA-bulk tile
//                       staging, warp multi-split ranking, windowed decoupled
//                       look-back, smem reorder, next pass's histogram
//                       (bitwise_sort_order / key_value_sort primitives.py:23-40)
//   K3   k_unique       adjacent-compare head flags + decoupled look-back scan,
//                       unique-row compaction, bucketed (org, new_idx) pairs
//                       (pipeline.py:72-113, primitives.py:43-69)
//   K3b  k_map_fill     map[org] = new_idx from the bucket-major pairs
//   K4   k_remap        out_idx = map[idx] (remap_elements pipeline.py:116-130)
//   gen  k_gen_lattice  synthetic bench input (oracle/lattice.py recipe)
//
// Data layout in HBM: a row is W = D+1 uint32 words -- the D key words of the
// (cleaned) vertex followed by its original index.  Rows are AoS so one tile
// of rows is one contiguous byte range, moved into shared memory with a
// single cp.async.bulk.  Key order is the reference's: raw unsigned words,
// component 0 most significant, so LSD pass p sorts byte (p % 4) of
// component D-1-p/4, pass 0 first.
#pragma once

#include "../../include/remesh_b200.h"
#include "rmx_common.cuh"

namespace rmx {

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;

// ---------------------------------------------------------------------------
// Plan layout (uint32 words, lives in the workspace):
//   [0] buffer holding the final sorted rows   [1] executed passes
//   [2] first executed pass                    [3] first pass needs k_first_hist
//   [4 + p]            pass p executes (digit not constant)
//   [4 + P + p]        source buffer of pass p
//   [4 + 2P + p]       next executed pass after p (P = none)
__host__ __device__ inline size_t plan_words(int P) { return 4 + 3 * static_cast<size_t>(P); }

// ---------------------------------------------------------------------------
// K1: mark used vertices; any index >= n_vtx sets the status bit.
struct MarkArgs {
    const uint32_t* idx;
    uint64_t n_idx;
    uint64_t n_vtx;
    uint8_t* flags;
    uint32_t* status;
    int vec;  // idx 16-byte aligned
};

__global__ void __launch_bounds__(kBlock) k_mark(MarkArgs a) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const uint64_t gtid = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    bool bad = false;
    uint64_t done = 0;
    if (a.vec) {
        const uint64_t n4 = a.n_idx >> 2;
        const uint4* i4 = reinterpret_cast<const uint4*>(a.idx);
        for (uint64_t i = gtid; i < n4; i += stride) {
            const uint4 v = __ldcs(i4 + i);
            const uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (x[k] < a.n_vtx) a.flags[x[k]] = 1;
                else bad = true;
            }
        }
        done = n4 << 2;
    }
    for (uint64_t i = done + gtid; i < a.n_idx; i += stride) {
        const uint32_t x = __ldcs(a.idx + i);
        if (x < a.n_vtx) a.flags[x] = 1;
        else bad = true;
    }
    if (__any_sync(kFull, bad) && (threadIdx.x & 31u) == 0u) atomicOr(a.status, RMX_STATUS_INDEX_OUT_OF_RANGE);
}

// ---------------------------------------------------------------------------
// K1b: cleaned AoS rows, the per-component "varying bits" masks that decide
// which digit passes execute, and the digit histograms of component D-1
// (passes 0..3: the first executed pass is almost always among them).
struct BuildArgs {
    const uint32_t* vtx;
    const uint8_t* flags;
    const uint32_t* idx;  // idx[0] is the replacement vertex (pipeline.py:148)
    uint32_t* rows;
    uint32_t* hist;       // [4D][256]; this kernel fills passes 0..3
    uint32_t* vary;       // [D]: OR over rows of (key ^ replacement key)
    const uint32_t* status;
    uint32_t n;
    int dim;
    int vec;              // vtx 16-byte aligned (4-row vector groups for D == 3)
};

// Run-length privatised histogram update: consecutive equal digits seen by a
// thread are added with one shared atomic (low-entropy mesh coordinates have
// long runs of identical bytes, which would otherwise serialise on one bank).
__device__ __forceinline__ void rl_push(uint32_t& st, uint32_t d, uint32_t* bins) {
    if ((st >> 8) != 0u && (st & 255u) == d) {
        st += 256u;
    } else {
        if ((st >> 8) != 0u) atomicAdd(bins + (st & 255u), st >> 8);
        st = 256u | d;
    }
}

template <int D_CT>
__global__ void __launch_bounds__(kBlock) k_build_rows(BuildArgs a) {
    const int D = D_CT > 0 ? D_CT : a.dim;
    const int W = D + 1;
    __shared__ uint32_t s_hist[4 * 256];
    __shared__ uint32_t s_vary[RMX_MAX_DIM];
    for (int i = threadIdx.x; i < 4 * 256; i += kBlock) s_hist[i] = 0u;
    if (threadIdx.x < RMX_MAX_DIM) s_vary[threadIdx.x] = 0u;
    __syncthreads();
    if (*a.status) return;  // uniform: written by K1, stable here

    const uint32_t r0 = a.idx[0];
    const uint32_t* repl = a.vtx + static_cast<size_t>(r0) * D;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const uint64_t start = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    uint32_t rl[4] = {0u, 0u, 0u, 0u};

    if constexpr (D_CT > 0) {
        uint32_t ref[D_CT], vor[D_CT];
#pragma unroll
        for (int c = 0; c < D_CT; ++c) {
            ref[c] = __ldg(repl + c);
            vor[c] = 0u;
        }
        auto emit = [&](uint64_t i, uint32_t (&k)[D_CT]) {
#pragma unroll
            for (int c = 0; c < D_CT; ++c) vor[c] |= k[c] ^ ref[c];
            const uint32_t last = k[D_CT - 1];
#pragma unroll
            for (int b = 0; b < 4; ++b) rl_push(rl[b], (last >> (8 * b)) & 255u, s_hist + b * 256);
            if constexpr (D_CT == 3) {
                reinterpret_cast<uint4*>(a.rows)[i] = make_uint4(k[0], k[1], k[2], static_cast<uint32_t>(i));
            } else {
                uint32_t* dst = a.rows + i * (D_CT + 1);
#pragma unroll
                for (int c = 0; c < D_CT; ++c) dst[c] = k[c];
                dst[D_CT] = static_cast<uint32_t>(i);
            }
        };
        uint64_t done = 0;
        if constexpr (D_CT == 3) {
            if (a.vec) {  // 4 rows = 3 x 16 B of vertex words + one 32-bit flag word
                const uint64_t ng = a.n >> 2;
                const uint4* v4 = reinterpret_cast<const uint4*>(a.vtx);
                const uint32_t* f4 = reinterpret_cast<const uint32_t*>(a.flags);
                for (uint64_t g = start; g < ng; g += stride) {
                    const uint4 x = __ldcs(v4 + 3 * g), y = __ldcs(v4 + 3 * g + 1), z = __ldcs(v4 + 3 * g + 2);
                    const uint32_t f = __ldcs(f4 + g);
                    uint32_t k[4][3] = {{x.x, x.y, x.z}, {x.w, y.x, y.y}, {y.z, y.w, z.x}, {z.y, z.z, z.w}};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (((f >> (8 * j)) & 255u) == 0u) {
#pragma unroll
                            for (int c = 0; c < 3; ++c) k[j][c] = ref[c];
                        }
                        emit(4 * g + j, k[j]);
                    }
                }
                done = ng << 2;
            }
        }
        for (uint64_t i = done + start; i < a.n; i += stride) {
            const bool used = a.flags[i] != 0;
            uint32_t k[D_CT];
#pragma unroll
            for (int c = 0; c < D_CT; ++c) k[c] = __ldg(a.vtx + i * D_CT + c);
            if (!used) {
#pragma unroll
                for (int c = 0; c < D_CT; ++c) k[c] = ref[c];
            }
            emit(i, k);
        }
#pragma unroll
        for (int c = 0; c < D_CT; ++c) {
            const uint32_t v = __reduce_or_sync(kFull, vor[c]);
            if ((threadIdx.x & 31u) == 0u && v) atomicOr(s_vary + c, v);
        }
    } else {
        for (uint64_t i = start; i < a.n; i += stride) {
            const bool used = a.flags[i] != 0;
            const uint32_t* srow = used ? a.vtx + i * D : repl;
            uint32_t* dst = a.rows + i * W;
            for (int c = 0; c < D; ++c) {
                const uint32_t k = __ldg(srow + c);
                dst[c] = k;
                const uint32_t x = k ^ __ldg(repl + c);
                if (x) atomicOr(s_vary + c, x);
                if (c == D - 1)
                    for (int b = 0; b < 4; ++b) rl_push(rl[b], (k >> (8 * b)) & 255u, s_hist + b * 256);
            }
            dst[D] = static_cast<uint32_t>(i);
        }
    }
#pragma unroll
    for (int b = 0; b < 4; ++b)
        if ((rl[b] >> 8) != 0u) atomicAdd(s_hist + b * 256 + (rl[b] & 255u), rl[b] >> 8);
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * 256; i += kBlock)
        if (s_hist[i]) atomicAdd(a.hist + i, s_hist[i]);
    if (threadIdx.x < static_cast<unsigned>(D) && s_vary[threadIdx.x]) atomicOr(a.vary + threadIdx.x, s_vary[threadIdx.x]);
}

// ---------------------------------------------------------------------------
// plan: a pass executes iff its digit is not constant over all keys (some
// bit of that byte differs from the replacement key in some row); assign
// ping-pong buffers and chain each executed pass to the next one.
__global__ void k_plan(const uint32_t* vary, uint32_t* plan, int D, const uint32_t* status) {
    if (*status || threadIdx.x != 0) return;
    const int P = 4 * D;
    uint32_t cur = 0, executed = 0, first = static_cast<uint32_t>(P), prev = static_cast<uint32_t>(P);
    for (int p = 0; p < P; ++p) {
        const int comp = D - 1 - (p >> 2);
        const bool ex = ((vary[comp] >> (8 * (p & 3))) & 255u) != 0u;
        plan[4 + p] = ex ? 1u : 0u;
        plan[4 + P + p] = cur;
        plan[4 + 2 * P + p] = static_cast<uint32_t>(P);
        if (ex) {
            if (first == static_cast<uint32_t>(P)) first = p;
            if (prev != static_cast<uint32_t>(P)) plan[4 + 2 * P + prev] = p;
            prev = p;
            cur ^= 1u;
            ++executed;
        }
    }
    plan[0] = cur;
    plan[1] = executed;
    plan[2] = first;
    plan[3] = (first < static_cast<uint32_t>(P) && first >= 4u) ? 1u : 0u;  // histogram not made by K1b
}

// Histogram of the first executed pass when it lies outside component D-1
// (only then; exits immediately otherwise).
struct HistArgs {
    const uint32_t* rows;
    uint32_t* hist;
    const uint32_t* plan;
    const uint32_t* status;
    uint32_t n;
    int dim;
};

__global__ void __launch_bounds__(kBlock) k_first_hist(HistArgs a) {
    if (*a.status || a.plan[3] == 0u) return;
    __shared__ uint32_t s_h[256];
    s_h[threadIdx.x] = 0u;
    __syncthreads();
    const uint32_t p = a.plan[2];
    const int comp = a.dim - 1 - static_cast<int>(p >> 2);
    const int shift = 8 * static_cast<int>(p & 3u);
    const int W = a.dim + 1;
    uint32_t rl = 0u;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x; i < a.n;
         i += static_cast<uint64_t>(gridDim.x) * kBlock)
        rl_push(rl, (__ldcs(a.rows + i * W + comp) >> shift) & 255u, s_h);
    if ((rl >> 8) != 0u) atomicAdd(s_h + (rl & 255u), rl >> 8);
    __syncthreads();
    if (s_h[threadIdx.x]) atomicAdd(a.hist + p * 256 + threadIdx.x, s_h[threadIdx.x]);
}

// ---------------------------------------------------------------------------
// K2: one onesweep LSD pass.  Persistent CTAs take tile ids from an atomic
// counter (forward progress for the look-back).  Tile data arrives by TMA
// bulk copy.  PF = 1 double-buffers: the NEXT tile id is taken only after the
// current tile has published its inclusive prefix (taking it earlier would
// hold back that tile's aggregate and convoy the look-back of later tiles),
// and its copy overlaps the reorder + write-out of the current tile.
// REG = rows held in registers and reordered in place; otherwise a per-slot
// source index (u16) drives the write-out straight from the staged tile.
// Each pass also counts the digit of the next executed pass (>= 4), so the
// global histogram of that pass is complete when it starts.
struct SortArgs {
    uint32_t* rows0;
    uint32_t* rows1;
    const uint32_t* plan;
    uint32_t* hist;      // [P][256]
    uint64_t* desc;      // [ntiles][256] look-back descriptors (shared by all passes, epoch-tagged)
    uint32_t* counters;  // [P] tile-id counters
    const uint32_t* status;
    uint32_t n;
    uint32_t ntiles;
    int dim;
    int pass;
    int ablate;  // tuning only (results invalid): 1 no look-back wait, 2 no ranking, 4 no write-out
};

constexpr int kRankMatch = 0;   // warp multi-split with match.any
constexpr int kRankBallot = 1;  // warp multi-split with 8 ballots

template <int W_CT, int IPT, bool REG, int PF>
struct SortTraits {
    static constexpr int kTile = kBlock * IPT;
    static constexpr int kBufs = PF ? 2 : 1;
    static __host__ __device__ size_t smem_bytes(int W) {
        return static_cast<size_t>(kBufs) * kTile * W * 4 + (kWarps * 256 + 256 * 3 + kWarps + 8) * 4 + 16 +
               (REG ? 0 : kTile * 2);
    }
};

template <int W_CT>
__device__ __forceinline__ uint32_t pick_word(const uint32_t* reg, int comp) {
    uint32_t k = reg[0];
#pragma unroll
    for (int c = 1; c < W_CT - 1; ++c) k = (comp == c) ? reg[c] : k;
    return k;
}

template <int W_CT, int IPT, int RANK, bool REG, int PF>
__global__ void __launch_bounds__(kBlock, REG ? 2 : 3) k_sort_pass(SortArgs a) {
    using T = SortTraits<W_CT, IPT, REG, PF>;
    constexpr int TILE = T::kTile;
    static_assert(!REG || W_CT > 0, "register rows need a compile-time width");
    const int W = W_CT > 0 ? W_CT : a.dim + 1;
    const int P = 4 * a.dim;
    if (*a.status) return;
    const uint32_t* plan = a.plan;
    if (plan[4 + a.pass] == 0u) return;  // constant digit: nothing moves
    const uint32_t src = plan[4 + P + a.pass];
    const uint32_t* __restrict__ in = src ? a.rows1 : a.rows0;
    uint32_t* __restrict__ out = src ? a.rows0 : a.rows1;
    const int comp = a.dim - 1 - (a.pass >> 2);
    const int shift = 8 * (a.pass & 3);
    const uint32_t epoch = static_cast<uint32_t>(a.pass) + 1u;
    const int nxt = static_cast<int>(plan[4 + 2 * P + a.pass]);
    // passes 0..3 are counted by K1b; later ones by the pass before them
    const bool count_next = nxt < P && nxt >= 4;
    const int ncomp = count_next ? a.dim - 1 - (nxt >> 2) : 0;
    const int nshift = 8 * (nxt & 3);
    uint32_t* ctr = a.counters + a.pass;

    extern __shared__ __align__(128) uint32_t smem[];
    const size_t tw = static_cast<size_t>(TILE) * W;
    uint32_t* s_buf = smem;                           // [kBufs][TILE * W]
    uint32_t* s_whist = smem + T::kBufs * tw;         // [warp][256]
    uint32_t* s_offs = s_whist + kWarps * 256;        // global exclusive digit starts
    uint32_t* s_gdst = s_offs + 256;                  // global row of tile slot 0, per digit
    uint32_t* s_hnext = s_gdst + 256;                 // histogram of the next executed pass
    uint32_t* s_warp = s_hnext + 256;
    uint32_t* s_misc = s_warp + kWarps;
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_misc + 8);
    uint16_t* s_src = reinterpret_cast<uint16_t*>(s_bar + 2);

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    auto tile_rows = [&](uint32_t t) { return min(static_cast<uint32_t>(TILE), a.n - t * static_cast<uint32_t>(TILE)); };
    auto load_tile = [&](uint32_t t, uint32_t buf) {
        stage_tile(s_buf + buf * tw, in + static_cast<size_t>(t) * TILE * W, tile_rows(t) * W * 4u, s_bar + buf);
    };

    if (tid == 0) {
        mbar_init(s_bar, 1);
        mbar_init(s_bar + 1, 1);
        fence_mbar_init();
        if (PF) {
            const uint32_t t0 = atomicAdd(ctr, 1u);
            s_misc[0] = t0;
            if (t0 < a.ntiles) load_tile(t0, 0);
        }
    }
    {
        uint32_t tot;
        const uint32_t h = a.hist[a.pass * 256 + tid];
        s_offs[tid] = block_exclusive_scan<kWarps>(h, s_warp, tot);
        s_hnext[tid] = 0u;
    }
    __syncthreads();
    uint32_t tile = PF ? s_misc[0] : 0u;
    for (uint32_t it = 0;; ++it) {
        const uint32_t b = PF ? (it & 1u) : 0u;
        uint32_t* s_cur = s_buf + b * tw;
        if (!PF && tid == 0) {
            const uint32_t t = atomicAdd(ctr, 1u);
            s_misc[0] = t;
            if (t < a.ntiles) load_tile(t, 0);
        }
        for (int i = tid; i < kWarps * 256; i += kBlock) s_whist[i] = 0u;
        __syncthreads();
        if (!PF) tile = s_misc[0];
        if (tile >= a.ntiles) break;
        const uint32_t tile_n = tile_rows(tile);
        mbar_wait(s_bar + b, PF ? ((it >> 1) & 1u) : (it & 1u));

        // ---- stable warp-level ranking: warp w owns rows [w*32*IPT, (w+1)*32*IPT).
        // Digits and peer masks of all IPT rounds are computed first (independent,
        // so the match latencies overlap); only the short per-round counter
        // read-modify-write chain is serial.
        uint32_t* wh = s_whist + warp * 256;
        uint32_t pk[IPT];  // digit, then digit << 16 | rank within the warp's rows of that digit
        uint32_t pm[IPT];  // peers (lanes of this round with the same digit)
        uint32_t reg[REG ? IPT * W_CT : 1];
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
            const bool valid = p < tile_n;
            uint32_t d = 256u;  // sentinel for rows past the end of the last tile
            if (valid) {
                uint32_t key, nkey = 0;
                if constexpr (W_CT == 4) {
                    const uint4 v = reinterpret_cast<const uint4*>(s_cur)[p];
                    if constexpr (REG) {
                        reg[r * 4 + 0] = v.x;
                        reg[r * 4 + 1] = v.y;
                        reg[r * 4 + 2] = v.z;
                        reg[r * 4 + 3] = v.w;
                    }
                    key = comp == 0 ? v.x : (comp == 1 ? v.y : v.z);
                    if (count_next) nkey = ncomp == 0 ? v.x : (ncomp == 1 ? v.y : v.z);
                } else if constexpr (REG) {
#pragma unroll
                    for (int c = 0; c < W_CT; ++c) reg[r * W_CT + c] = s_cur[p * W_CT + c];
                    key = pick_word<W_CT>(reg + r * W_CT, comp);
                    if (count_next) nkey = pick_word<W_CT>(reg + r * W_CT, ncomp);
                } else {
                    key = s_cur[static_cast<size_t>(p) * W + comp];
                    if (count_next) nkey = s_cur[static_cast<size_t>(p) * W + ncomp];
                }
                d = (key >> shift) & 255u;
                if (count_next) atomicAdd(s_hnext + ((nkey >> nshift) & 255u), 1u);
            }
            pk[r] = d;
        }
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t d = pk[r];
            if (a.ablate & 2) {
                pm[r] = 1u << lane;
                continue;
            }
            if constexpr (RANK == kRankBallot) {
                uint32_t peers = kFull;
#pragma unroll
                for (int bit = 0; bit < 9; ++bit) {
                    const uint32_t bb = __ballot_sync(kFull, (d >> bit) & 1u);
                    peers &= ((d >> bit) & 1u) ? bb : ~bb;
                }
                pm[r] = peers;
            } else {
                pm[r] = __match_any_sync(kFull, d);
            }
        }
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t d = pk[r];
            const uint32_t peers = pm[r];
            uint32_t before = 0;
            if (d < 256u) before = wh[d];
            __syncwarp();
            if (d < 256u && (peers & lanemask_lt()) == 0u) wh[d] = before + __popc(peers);
            __syncwarp();
            pk[r] = (d << 16) | (before + __popc(peers & lanemask_lt()));
        }
        __syncthreads();

        // ---- per digit (thread d): tile count, publish, local start, windowed look-back
        {
            const uint32_t d = tid;
            uint32_t wc[kWarps];
            uint32_t cnt = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                wc[w] = s_whist[w * 256 + d];
                cnt += wc[w];
            }
            uint64_t* mine = a.desc + static_cast<size_t>(tile) * 256 + d;
            st_relaxed(mine, pack_desc(epoch, tile == 0 ? kPrefix : kAggregate, cnt));
            uint32_t tot;
            const uint32_t start = block_exclusive_scan<kWarps>(cnt, s_warp, tot);
            uint32_t run = start;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                s_whist[w * 256 + d] = run;  // slot of this warp's first row with digit d
                run += wc[w];
            }
            uint32_t excl = 0;
            if (tile > 0 && !(a.ablate & 1)) {
                int64_t t = static_cast<int64_t>(tile) - 1;
                for (;;) {
                    constexpr int LB = 4;
                    uint64_t v[LB];
#pragma unroll
                    for (int j = 0; j < LB; ++j)
                        v[j] = (t - j >= 0) ? ld_relaxed(a.desc + static_cast<size_t>(t - j) * 256 + d)
                                            : pack_desc(epoch, kPrefix, 0u);
                    bool done = false;
#pragma unroll
                    for (int j = 0; j < LB; ++j) {
                        if (!done) {
                            while (desc_epoch(v[j]) != epoch || desc_flag(v[j]) == 0u) {
                                __nanosleep(20);
                                v[j] = ld_relaxed(a.desc + static_cast<size_t>(t - j) * 256 + d);
                            }
                            excl += desc_value(v[j]);
                            done = desc_flag(v[j]) == kPrefix;
                        }
                    }
                    if (done) break;
                    t -= LB;
                }
                st_relaxed(mine, pack_desc(epoch, kPrefix, excl + cnt));
            }
            s_gdst[d] = s_offs[d] + excl - start;  // mod 2^32; + tile slot gives the global row
        }
        if (PF && tid == 0) {  // prefix published: now take the next tile and start its copy
            const uint32_t t = atomicAdd(ctr, 1u);
            s_misc[1] = t;
            if (t < a.ntiles) load_tile(t, b ^ 1u);
        }
        __syncthreads();

        // ---- reorder into digit order (in place from registers, or via a slot -> row index)
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
            if (p < tile_n) {
                const uint32_t slot = s_whist[warp * 256 + (pk[r] >> 16)] + (pk[r] & 0xFFFFu);
                if constexpr (REG) {
                    if constexpr (W_CT == 4) {
                        reinterpret_cast<uint4*>(s_cur)[slot] =
                            make_uint4(reg[r * 4 + 0], reg[r * 4 + 1], reg[r * 4 + 2], reg[r * 4 + 3]);
                    } else {
#pragma unroll
                        for (int c = 0; c < W_CT; ++c) s_cur[slot * W_CT + c] = reg[r * W_CT + c];
                    }
                } else {
                    s_src[slot] = static_cast<uint16_t>(p);
                }
            }
        }
        __syncthreads();

        // ---- coalesced write-out: consecutive slots of one digit are consecutive rows
        if (a.ablate & 4) {
        } else if constexpr (W_CT == 4) {
            const uint4* s4 = reinterpret_cast<const uint4*>(s_cur);
            uint4* o4 = reinterpret_cast<uint4*>(out);
            constexpr int U = 4;  // independent LDS -> LDS -> STG chains in flight per thread
            for (uint32_t q0 = tid; q0 < tile_n; q0 += U * kBlock) {
                uint4 v[U];
                uint32_t dst[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t q = q0 + u * kBlock;
                    if (q < tile_n) v[u] = REG ? s4[q] : s4[s_src[q]];
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t q = q0 + u * kBlock;
                    if (q < tile_n) {
                        const uint32_t key = comp == 0 ? v[u].x : (comp == 1 ? v[u].y : v[u].z);
                        dst[u] = s_gdst[(key >> shift) & 255u] + q;
                        if (a.ablate) dst[u] = min(dst[u], a.n - 1u);  // keep ablated runs in bounds
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t q = q0 + u * kBlock;
                    if (q < tile_n) o4[dst[u]] = v[u];
                }
            }
        } else {
            const uint32_t nw = tile_n * W;
            for (uint32_t q = tid; q < nw; q += kBlock) {
                const uint32_t slot = q / W;
                const uint32_t c = q - slot * W;
                const size_t p = REG ? slot : s_src[slot];
                const uint32_t d = (s_cur[p * W + comp] >> shift) & 255u;
                out[static_cast<size_t>(s_gdst[d] + slot) * W + c] = s_cur[p * W + c];
            }
        }
        if (PF) tile = s_misc[1];
        __syncthreads();
    }
    if (count_next && s_hnext[tid]) atomicAdd(a.hist + nxt * 256 + tid, s_hnext[tid]);
}

// ---------------------------------------------------------------------------
// K3: head flags, decoupled look-back scan, unique compaction, and the
// old->new pairs.  invert_permutation + remap (pipeline.py:103-130) need
// map[org_id[j]] = new_idx[j]: a random 4-byte scatter over V entries that
// costs ~35 B of DRAM traffic per row when done directly.  Instead each tile
// buckets its (org, new_idx) pairs by the high bits of org in shared memory
// and appends each bucket run to that bucket's contiguous region of a pair
// array (the free ping-pong row buffer); K3b then streams the pairs bucket
// by bucket, so its map stores stay inside an L2-resident window.
struct UniqueArgs {
    const uint32_t* rows0;
    const uint32_t* rows1;
    const uint32_t* plan;
    uint64_t* desc;     // [ntiles]
    uint32_t* counter;  // tile-id counter
    uint32_t* fill;     // [256] per-bucket append counters
    const uint32_t* status;
    uint32_t* out_vtx;  // [U][D]
    unsigned long long* count;
    uint32_t* sc_org;   // optional scratch outputs
    uint8_t* sc_nodup;
    uint32_t* sc_new;
    uint32_t* sc_perm;
    uint32_t n;
    uint32_t ntiles;
    int dim;
    int bucket_shift;   // bucket = org >> bucket_shift (<= 256 buckets)
};

template <int W_CT, int IPT>
struct UniqueTraits {
    static constexpr int kTile = kBlock * IPT;
    static __host__ __device__ size_t smem_bytes(int W) {
        return static_cast<size_t>(kTile) * W * 4 + static_cast<size_t>(kTile) * 8 + (64 + 4 * 256 + 2 * kWarps + 8) * 4 +
               16;
    }
};

template <int W_CT, int IPT>
__global__ void __launch_bounds__(kBlock) k_unique(UniqueArgs a) {
    using T = UniqueTraits<W_CT, IPT>;
    constexpr int TILE = T::kTile;
    const int D = W_CT > 0 ? W_CT - 1 : a.dim;
    const int W = D + 1;
    if (*a.status) return;
    const uint32_t* __restrict__ rows = a.plan[0] ? a.rows1 : a.rows0;
    uint2* __restrict__ pairs = reinterpret_cast<uint2*>(a.plan[0] ? const_cast<uint32_t*>(a.rows0)
                                                                    : const_cast<uint32_t*>(a.rows1));

    extern __shared__ __align__(128) uint32_t smem[];
    const size_t tw = static_cast<size_t>(TILE) * W;
    uint32_t* s_rows = smem;
    uint2* s_pairs = reinterpret_cast<uint2*>(smem + tw);     // tile pairs, bucket order
    uint32_t* s_prev = smem + tw + 2 * TILE;                   // up to 64 words
    uint32_t* s_bcnt = s_prev + 64;                            // per-bucket count in tile
    uint32_t* s_bcur = s_bcnt + 256;                           // running local slot per bucket
    uint32_t* s_bglob = s_bcur + 256;                          // pair index of local slot 0, per bucket
    uint32_t* s_bsave = s_bglob + 256;
    uint32_t* s_warp = s_bsave + 256;
    uint32_t* s_misc = s_warp + 2 * kWarps;
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_misc + 8);

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const int bs = a.bucket_shift;
    if (tid == 0) {
        mbar_init(s_bar, 1);
        fence_mbar_init();
    }
    for (uint32_t it = 0;; ++it) {
        if (tid == 0) {
            const uint32_t t = atomicAdd(a.counter, 1u);
            s_misc[0] = t;
            if (t < a.ntiles) {
                const uint32_t tn = min(static_cast<uint32_t>(TILE), a.n - t * static_cast<uint32_t>(TILE));
                stage_tile(s_rows, rows + static_cast<size_t>(t) * TILE * W, tn * W * 4u, s_bar);
            }
        }
        s_bcnt[tid] = 0u;
        __syncthreads();
        const uint32_t tile = s_misc[0];
        if (tile >= a.ntiles) break;
        const uint32_t base = tile * static_cast<uint32_t>(TILE);
        const uint32_t tile_n = min(static_cast<uint32_t>(TILE), a.n - base);
        if (tile > 0 && tid < static_cast<uint32_t>(D)) s_prev[tid] = rows[static_cast<size_t>(base - 1) * W + tid];
        __syncthreads();
        mbar_wait(s_bar, it & 1u);

        // ---- phase 1: head flags (warp-striped rows), per-warp totals, bucket counts
        uint32_t bal[IPT];
        uint32_t wtotal = 0;
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
            bool head = false;
            if (p < tile_n) {
                const uint32_t* cur = s_rows + static_cast<size_t>(p) * W;
                if (base + p == 0u) {
                    head = true;
                } else {
                    const uint32_t* prv = p ? cur - W : s_prev;
                    if constexpr (W_CT > 0) {
#pragma unroll
                        for (int c = 0; c < W_CT - 1; ++c) head |= cur[c] != prv[c];
                    } else {
                        for (int c = 0; c < D; ++c) head |= cur[c] != prv[c];
                    }
                }
                atomicAdd(s_bcnt + (cur[D] >> bs), 1u);
            }
            bal[r] = __ballot_sync(kFull, head);
            wtotal += __popc(bal[r]);
        }
        if (lane == 0) s_warp[warp] = wtotal;
        __syncthreads();
        uint32_t wexcl = 0, ttotal = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t t = s_warp[w];
            wexcl += (static_cast<uint32_t>(w) < warp) ? t : 0u;
            ttotal += t;
        }
        // bucket b (thread b): local start, and append space in the global pair array
        {
            const uint32_t cnt = s_bcnt[tid];
            uint32_t tot;
            const uint32_t start = block_exclusive_scan<kWarps>(cnt, s_warp + kWarps, tot);
            s_bcur[tid] = start;
            s_bsave[tid] = start;
            if (cnt) s_bglob[tid] = (tid << bs) + atomicAdd(a.fill + tid, cnt) - start;
        }

        // ---- decoupled look-back over tiles (warp 0, 32 predecessors per window;
        // waits only for the descriptors up to the nearest inclusive prefix)
        if (warp == 0) {
            uint64_t* mine = a.desc + tile;
            uint32_t excl = 0;
            if (tile == 0) {
                if (lane == 0) st_relaxed(mine, pack_desc(1u, kPrefix, ttotal));
            } else {
                if (lane == 0) st_relaxed(mine, pack_desc(1u, kAggregate, ttotal));
                int64_t hi = static_cast<int64_t>(tile) - 1;
                for (;;) {
                    const int64_t t = hi - static_cast<int64_t>(lane);
                    uint64_t dd = t >= 0 ? ld_relaxed(a.desc + t) : pack_desc(1u, kPrefix, 0u);
                    bool done = false;
                    for (;;) {
                        const bool valid = desc_epoch(dd) == 1u && desc_flag(dd) != 0u;
                        const uint32_t vm = __ballot_sync(kFull, valid);
                        const uint32_t pm = __ballot_sync(kFull, valid && desc_flag(dd) == kPrefix);
                        const uint32_t need = pm ? (((pm & (0u - pm)) << 1) - 1u) : kFull;
                        if ((vm & need) == need) {
                            excl += warp_sum(((need >> lane) & 1u) ? desc_value(dd) : 0u);
                            done = pm != 0u;
                            break;
                        }
                        if (!valid) {
                            __nanosleep(20);
                            dd = ld_relaxed(a.desc + t);
                        }
                    }
                    if (done) break;
                    hi -= 32;
                }
                if (lane == 0) st_relaxed(mine, pack_desc(1u, kPrefix, excl + ttotal));
            }
            if (lane == 0) s_misc[2] = excl;
        }
        __syncthreads();
        const uint32_t tprefix = s_misc[2];
        if (tid == 0 && tile == a.ntiles - 1) *a.count = static_cast<unsigned long long>(tprefix) + ttotal;

        // ---- phase 2: new index per slot, bucketed pairs, unique rows out
        uint32_t running = tprefix + wexcl;
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
            if (p < tile_n) {
                const uint32_t* row = s_rows + static_cast<size_t>(p) * W;
                const uint32_t nidx = running + __popc(bal[r] & lanemask_le()) - 1u;
                const uint32_t org = row[D];
                s_pairs[atomicAdd(s_bcur + (org >> bs), 1u)] = make_uint2(org, nidx);
                const bool head = (bal[r] >> lane) & 1u;
                if (head) {
                    uint32_t* dst = a.out_vtx + static_cast<size_t>(nidx) * D;
                    for (int c = 0; c < D; ++c) dst[c] = row[c];
                }
                if (a.sc_org) a.sc_org[base + p] = org;
                if (a.sc_nodup) a.sc_nodup[base + p] = head ? 1 : 0;
                if (a.sc_new) a.sc_new[base + p] = nidx;
                if (a.sc_perm) a.sc_perm[org] = base + p;
            }
            running += __popc(bal[r]);
        }
        __syncthreads();
        // ---- bucket runs out: consecutive slots of one bucket are consecutive pairs
        for (uint32_t q = tid; q < tile_n; q += kBlock) {
            const uint2 pr = s_pairs[q];
            pairs[s_bglob[pr.x >> bs] + q] = pr;
        }
        __syncthreads();
    }
}

// K3b: map[org] = new_idx from the bucket-major pair array (streaming reads;
// the stores of concurrently running CTAs fall in one or two buckets, i.e. an
// L2-resident window of map, so partial sectors merge before write-back).
__global__ void __launch_bounds__(kBlock) k_map_fill(const uint32_t* plan, const uint32_t* rows0,
                                                      const uint32_t* rows1, uint32_t* map, uint32_t n,
                                                      const uint32_t* status) {
    if (*status) return;
    const uint4* pairs = reinterpret_cast<const uint4*>(plan[0] ? rows0 : rows1);
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;  // two pairs per thread
    if (2 * i + 1 < n) {
        const uint4 v = __ldcs(pairs + i);
        map[v.x] = v.y;
        map[v.z] = v.w;
    } else if (2 * i < n) {
        const uint2 v = reinterpret_cast<const uint2*>(pairs)[2 * i];
        map[v.x] = v.y;
    }
}

// ---------------------------------------------------------------------------
// K4: out_idx[k] = map[idx[k]].
struct RemapArgs {
    const uint32_t* idx;
    const uint32_t* map;
    uint32_t* out;
    uint64_t n_idx;
    const uint32_t* status;
    int vec;
};

__global__ void __launch_bounds__(kBlock) k_remap(RemapArgs a) {
    if (*a.status) return;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const uint64_t gtid = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    uint64_t done = 0;
    if (a.vec) {
        const uint64_t n4 = a.n_idx >> 2;
        const uint4* i4 = reinterpret_cast<const uint4*>(a.idx);
        uint4* o4 = reinterpret_cast<uint4*>(a.out);
        for (uint64_t i = gtid; i < n4; i += stride) {
            const uint4 v = __ldcs(i4 + i);
            uint4 o;
            o.x = __ldg(a.map + v.x);
            o.y = __ldg(a.map + v.y);
            o.z = __ldg(a.map + v.z);
            o.w = __ldg(a.map + v.w);
            __stcs(o4 + i, o);
        }
        done = n4 << 2;
    }
    for (uint64_t i = done + gtid; i < a.n_idx; i += stride) a.out[i] = __ldg(a.map + __ldcs(a.idx + i));
}

// ---------------------------------------------------------------------------
// Synthetic lattice soups (bit-identical to oracle/lattice.py).
__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct GenArgs {
    int kind;  // 0 tri, 1 tet
    uint32_t nx, ny, nz;
    uint64_t n_elem;  // total lattice elements (permutation domain)
    uint64_t take;    // elements written
    uint64_t n_unused;
    uint32_t half;
    uint64_t mask;
    uint64_t keys[4];
    uint64_t useed;
    uint32_t* vtx;
    uint32_t* idx;
};

__device__ __forceinline__ uint64_t feistel(uint64_t v, const GenArgs& g) {
    uint64_t left = v >> g.half, right = v & g.mask;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const uint64_t f = (splitmix64(right ^ g.keys[r]) >> 7) & g.mask;
        const uint64_t nl = right;
        right = left ^ f;
        left = nl;
    }
    return (left << g.half) | right;
}

__global__ void __launch_bounds__(kBlock) k_gen_lattice(GenArgs g) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const int K = g.kind == 0 ? 3 : 4;
    const int D = K;
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x; e < g.take; e += stride) {
        uint64_t t = feistel(e, g);
        while (t >= g.n_elem) t = feistel(t, g);
        const uint64_t u0 = (e * g.n_unused) / g.n_elem;
        const uint64_t u1 = ((e + 1) * g.n_unused) / g.n_elem;
        const uint64_t base = e * K + u0;
        int pts[4][3];
        if (g.kind == 0) {
            const uint64_t q = t >> 1;
            const int h = static_cast<int>(t & 1);
            const int qi = static_cast<int>(q / g.ny), qj = static_cast<int>(q % g.ny);
            pts[0][0] = qi;     pts[0][1] = qj;
            pts[1][0] = qi + 1; pts[1][1] = h ? qj + 1 : qj;
            pts[2][0] = h ? qi : qi + 1; pts[2][1] = qj + 1;
        } else {
            const uint64_t c = t / 6;
            const int s = static_cast<int>(t % 6);
            const int ci = static_cast<int>(c / (static_cast<uint64_t>(g.ny) * g.nz));
            const int cj = static_cast<int>((c / g.nz) % g.ny);
            const int ck = static_cast<int>(c % g.nz);
            const int kuhn[6][2] = {{0, 1}, {0, 2}, {1, 0}, {1, 2}, {2, 0}, {2, 1}};
            int v[3] = {ci, cj, ck};
            for (int x = 0; x < 3; ++x) pts[0][x] = v[x];
            v[kuhn[s][0]] += 1;
            for (int x = 0; x < 3; ++x) pts[1][x] = v[x];
            v[kuhn[s][1]] += 1;
            for (int x = 0; x < 3; ++x) pts[2][x] = v[x];
            for (int x = 0; x < 3; ++x) pts[3][x] = pts[0][x] + 1;
        }
        for (int s = 0; s < K; ++s) {
            uint32_t* row = g.vtx + (base + s) * D;
            const int i = pts[s][0], j = pts[s][1];
            if (g.kind == 0) {
                row[0] = __float_as_uint(__fmul_rn(static_cast<float>(i), 0.5f));
                row[1] = __float_as_uint(__fmul_rn(static_cast<float>(j), 0.5f));
                row[2] = __float_as_uint(__fmul_rn(static_cast<float>((7 * i + 13 * j) % 64), 0.25f));
            } else {
                const int k = pts[s][2];
                row[0] = __float_as_uint(__fmul_rn(static_cast<float>(i), 0.5f));
                row[1] = __float_as_uint(__fmul_rn(static_cast<float>(j), 0.5f));
                row[2] = __float_as_uint(__fmul_rn(static_cast<float>(k), 0.5f));
                row[3] = __float_as_uint(__fmul_rn(static_cast<float>((3 * i + 5 * j + 7 * k) % 97), 0.125f));
            }
            g.idx[e * K + s] = static_cast<uint32_t>(base + s);
        }
        for (uint64_t o = u0; o < u1; ++o) {
            uint32_t* row = g.vtx + (base + K + (o - u0)) * D;
            for (int c = 0; c < D; ++c) {
                const uint64_t h = splitmix64((o * D + c) ^ g.useed);
                const uint64_t expo = (0x7Full + ((h >> 32) % 10ull)) << 23;
                row[c] = static_cast<uint32_t>((h & 0x807FFFFFull) | expo);
            }
        }
    }
}

}  // namespace rmx
