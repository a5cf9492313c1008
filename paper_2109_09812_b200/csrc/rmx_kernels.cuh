// rmx_kernels.cuh -- the sm_100a kernels of the re-indexing pipeline.
//
//   K1   k_mark         isUsed scatter over the index buffer + range check
//                       (reference mark_used pipeline.py:41-51, require_valid mesh.py:103-105)
//   K1b  k_build_rows   unused -> replacement, AoS (key words, origin) rows, and
//                       the 8-bit digit histograms of every LSD pass
//                       (overwrite_unused pipeline.py:54-63, fill_sequence primitives.py:16-20)
//   plan k_plan         digit-pass skipping, ping-pong schedule, global digit offsets
//   K2   k_sort_pass    one onesweep LSD pass: TMA-bulk tile staging, warp
//                       match_any ranking, decoupled look-back, smem reorder
//                       (bitwise_sort_order / key_value_sort primitives.py:23-40)
//   K3   k_unique       adjacent-compare head flags + decoupled look-back scan,
//                       old->new map scatter and unique-row compaction
//                       (pipeline.py:72-113, primitives.py:43-69)
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

#include "rmx_common.cuh"

namespace rmx {

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;

// ---------------------------------------------------------------------------
// Plan layout (uint32 words, lives in the workspace):
//   [0] buffer holding the final sorted rows   [1] executed passes
//   [4 + p]            pass p executes (digit not constant)
//   [4 + P + p]        source buffer of pass p
//   [4 + 2P + 256p + d] global exclusive start of digit d in pass p
__host__ __device__ inline size_t plan_words(int P) { return 4 + 2 * static_cast<size_t>(P) + 256 * static_cast<size_t>(P); }

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
// K1b: cleaned rows + all digit histograms.
struct BuildArgs {
    const uint32_t* vtx;
    const uint8_t* flags;
    const uint32_t* idx;  // idx[0] is the replacement vertex (pipeline.py:148)
    uint32_t* rows;
    uint32_t* hist;       // [4D][256]
    const uint32_t* status;
    uint32_t n;
    int dim;
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
    const int P = 4 * D;
    extern __shared__ __align__(16) uint32_t s_hist[];  // P * 256
    for (int i = threadIdx.x; i < P * 256; i += kBlock) s_hist[i] = 0u;
    __syncthreads();
    if (*a.status) return;  // uniform: written by K1, stable here

    const uint32_t r0 = a.idx[0];
    const uint32_t* repl = a.vtx + static_cast<size_t>(r0) * D;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const uint64_t start = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;

    if constexpr (D_CT > 0) {
        uint32_t rl[4 * D_CT];
#pragma unroll
        for (int p = 0; p < 4 * D_CT; ++p) rl[p] = 0u;
        for (uint64_t i = start; i < a.n; i += stride) {
            const bool used = a.flags[i] != 0;
            const uint32_t* srow = used ? a.vtx + i * D_CT : repl;
            uint32_t k[D_CT];
#pragma unroll
            for (int c = 0; c < D_CT; ++c) k[c] = __ldg(srow + c);
            if constexpr (D_CT == 3) {
                reinterpret_cast<uint4*>(a.rows)[i] = make_uint4(k[0], k[1], k[2], static_cast<uint32_t>(i));
            } else {
                uint32_t* dst = a.rows + i * (D_CT + 1);
#pragma unroll
                for (int c = 0; c < D_CT; ++c) dst[c] = k[c];
                dst[D_CT] = static_cast<uint32_t>(i);
            }
#pragma unroll
            for (int p = 0; p < 4 * D_CT; ++p) {
                const int c = D_CT - 1 - (p >> 2);
                rl_push(rl[p], (k[c] >> (8 * (p & 3))) & 255u, s_hist + p * 256);
            }
        }
#pragma unroll
        for (int p = 0; p < 4 * D_CT; ++p)
            if ((rl[p] >> 8) != 0u) atomicAdd(s_hist + p * 256 + (rl[p] & 255u), rl[p] >> 8);
    } else {
        for (uint64_t i = start; i < a.n; i += stride) {
            const bool used = a.flags[i] != 0;
            const uint32_t* srow = used ? a.vtx + i * D : repl;
            uint32_t* dst = a.rows + i * W;
            for (int c = 0; c < D; ++c) {
                const uint32_t k = __ldg(srow + c);
                dst[c] = k;
                const int pbase = 4 * (D - 1 - c);
#pragma unroll
                for (int b = 0; b < 4; ++b) atomicAdd(s_hist + (pbase + b) * 256 + ((k >> (8 * b)) & 255u), 1u);
            }
            dst[D] = static_cast<uint32_t>(i);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < P * 256; i += kBlock)
        if (s_hist[i]) atomicAdd(a.hist + i, s_hist[i]);
}

// ---------------------------------------------------------------------------
// plan: skip passes whose digit is constant, assign ping-pong buffers, and
// exclusive-scan each digit histogram into global bucket starts.
__global__ void __launch_bounds__(kBlock) k_plan(const uint32_t* hist, uint32_t* plan, int P, uint32_t n,
                                                  const uint32_t* status) {
    if (*status) return;
    __shared__ uint32_t s_warp[kWarps];
    uint32_t cur = 0, executed = 0;
    for (int p = 0; p < P; ++p) {
        const uint32_t c = hist[p * 256 + threadIdx.x];
        const int constant = __syncthreads_or(c == n);
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan<kWarps>(c, s_warp, tot);
        plan[4 + 2 * P + p * 256 + threadIdx.x] = ex;
        if (threadIdx.x == 0) {
            plan[4 + p] = constant ? 0u : 1u;
            plan[4 + P + p] = cur;
        }
        if (!constant) {
            cur ^= 1u;
            ++executed;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        plan[0] = cur;
        plan[1] = executed;
    }
}

// ---------------------------------------------------------------------------
// K2: one onesweep LSD pass (persistent CTAs, dynamic tile ids).
struct SortArgs {
    uint32_t* rows0;
    uint32_t* rows1;
    const uint32_t* plan;
    uint64_t* desc;      // [ntiles][256] look-back descriptors (shared by all passes, epoch-tagged)
    uint32_t* counters;  // [P] tile-id counters
    const uint32_t* status;
    uint32_t n;
    uint32_t ntiles;
    int dim;
    int pass;
};

template <int W_CT, int IPT>
struct SortTraits {
    static constexpr int kTile = kBlock * IPT;
    // W_CT > 0: rows are held in registers and reordered in place (one buffer);
    // generic W: separate input and output staging buffers.
    static constexpr int kBuffers = W_CT > 0 ? 1 : 2;
    static __host__ __device__ size_t smem_bytes(int W) {
        return static_cast<size_t>(kBuffers) * kTile * W * 4 + (kWarps * 256 + 512 + kWarps + 8) * 4 + 16;
    }
};

template <int W_CT, int IPT>
__global__ void __launch_bounds__(kBlock) k_sort_pass(SortArgs a) {
    using T = SortTraits<W_CT, IPT>;
    constexpr int TILE = T::kTile;
    const int W = W_CT > 0 ? W_CT : a.dim + 1;
    const int P = 4 * a.dim;
    if (*a.status) return;
    const uint32_t* plan = a.plan;
    if (plan[4 + a.pass] == 0u) return;  // constant digit: nothing moves
    const uint32_t src = plan[4 + P + a.pass];
    const uint32_t* __restrict__ in = src ? a.rows1 : a.rows0;
    uint32_t* __restrict__ out = src ? a.rows0 : a.rows1;
    const uint32_t* offs = plan + 4 + 2 * P + 256 * a.pass;
    const int comp = a.dim - 1 - (a.pass >> 2);
    const int shift = 8 * (a.pass & 3);
    const uint32_t epoch = static_cast<uint32_t>(a.pass) + 1u;

    extern __shared__ __align__(128) uint32_t smem[];
    uint32_t* s_in = smem;
    uint32_t* s_out = (W_CT > 0) ? s_in : s_in + static_cast<size_t>(TILE) * W;
    uint32_t* s_whist = s_out + static_cast<size_t>(TILE) * W;  // [warp][256]
    uint32_t* s_start = s_whist + kWarps * 256;                   // tile-local digit start
    uint32_t* s_gdst = s_start + 256;                             // global row of local slot 0, per digit
    uint32_t* s_warp = s_gdst + 256;
    uint32_t* s_misc = s_warp + kWarps;
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_misc + 8);

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    if (tid == 0) {
        mbar_init(s_bar, 1);
        fence_mbar_init();
    }
    __syncthreads();

    for (uint32_t iter = 0;; ++iter) {
        if (tid == 0) s_misc[0] = atomicAdd(a.counters + a.pass, 1u);
        for (int i = tid; i < kWarps * 256; i += kBlock) s_whist[i] = 0u;
        __syncthreads();
        const uint32_t tile = s_misc[0];
        if (tile >= a.ntiles) break;
        const uint32_t base = tile * static_cast<uint32_t>(TILE);
        const uint32_t tile_n = min(static_cast<uint32_t>(TILE), a.n - base);
        if (tid == 0) stage_tile(s_in, in + static_cast<size_t>(base) * W, tile_n * W * 4u, s_bar);
        mbar_wait(s_bar, iter & 1u);

        // ---- stable warp-level ranking: warp w owns rows [w*32*IPT, (w+1)*32*IPT)
        uint32_t* wh = s_whist + warp * 256;
        uint32_t rank[IPT];
        uint32_t dig[IPT];
        uint32_t reg[W_CT > 0 ? IPT * W_CT : 1];
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
            const bool valid = p < tile_n;
            uint32_t d = 0;
            if (valid) {
                d = (s_in[static_cast<size_t>(p) * W + comp] >> shift) & 255u;
                if constexpr (W_CT == 4) {
                    const uint4 v = reinterpret_cast<const uint4*>(s_in)[p];
                    reg[r * 4 + 0] = v.x;
                    reg[r * 4 + 1] = v.y;
                    reg[r * 4 + 2] = v.z;
                    reg[r * 4 + 3] = v.w;
                } else if constexpr (W_CT > 0) {
#pragma unroll
                    for (int c = 0; c < W_CT; ++c) reg[r * W_CT + c] = s_in[p * W_CT + c];
                }
            }
            const uint32_t vmask = __ballot_sync(kFull, valid);
            uint32_t peers = 0, before = 0;
            if (valid) {
                peers = __match_any_sync(vmask, d);
                before = wh[d];
            }
            __syncwarp();
            if (valid && (peers & lanemask_lt()) == 0u) wh[d] = before + __popc(peers);
            __syncwarp();
            rank[r] = before + __popc(peers & lanemask_lt());
            dig[r] = d;
        }
        __syncthreads();

        // ---- per digit: warp offsets, tile count, publish, local start, look-back
        {
            const uint32_t d = tid;
            uint32_t cnt = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const uint32_t c = s_whist[w * 256 + d];
                s_whist[w * 256 + d] = cnt;
                cnt += c;
            }
            uint64_t* mine = a.desc + static_cast<size_t>(tile) * 256 + d;
            st_relaxed(mine, pack_desc(epoch, tile == 0 ? kPrefix : kAggregate, cnt));
            uint32_t tot;
            const uint32_t start = block_exclusive_scan<kWarps>(cnt, s_warp, tot);
            s_start[d] = start;
            uint32_t excl = 0;
            if (tile > 0) {
                int64_t t = static_cast<int64_t>(tile) - 1;
                for (;;) {
                    const uint64_t dd = wait_desc(a.desc + static_cast<size_t>(t) * 256 + d, epoch);
                    excl += desc_value(dd);
                    if (desc_flag(dd) == kPrefix) break;
                    --t;
                }
                st_relaxed(mine, pack_desc(epoch, kPrefix, excl + cnt));
            }
            s_gdst[d] = offs[d] + excl - start;  // mod 2^32; + local slot gives the global row
        }
        __syncthreads();

        // ---- reorder the tile into digit order in shared memory
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
            if (p < tile_n) {
                const uint32_t d = dig[r];
                const uint32_t slot = s_start[d] + s_whist[warp * 256 + d] + rank[r];
                if constexpr (W_CT == 4) {
                    reinterpret_cast<uint4*>(s_out)[slot] =
                        make_uint4(reg[r * 4 + 0], reg[r * 4 + 1], reg[r * 4 + 2], reg[r * 4 + 3]);
                } else if constexpr (W_CT > 0) {
#pragma unroll
                    for (int c = 0; c < W_CT; ++c) s_out[slot * W_CT + c] = reg[r * W_CT + c];
                } else {
                    for (int c = 0; c < W; ++c) s_out[static_cast<size_t>(slot) * W + c] = s_in[static_cast<size_t>(p) * W + c];
                }
            }
        }
        __syncthreads();

        // ---- coalesced write-out: consecutive slots of one digit are consecutive rows
        if constexpr (W_CT == 4) {
            const uint4* s4 = reinterpret_cast<const uint4*>(s_out);
            uint4* o4 = reinterpret_cast<uint4*>(out);
            for (uint32_t p = tid; p < tile_n; p += kBlock) {
                const uint32_t d = (s_out[p * 4 + comp] >> shift) & 255u;
                o4[s_gdst[d] + p] = s4[p];
            }
        } else {
            const uint32_t nw = tile_n * W;
            for (uint32_t q = tid; q < nw; q += kBlock) {
                const uint32_t p = q / W;
                const uint32_t c = q - p * W;
                const uint32_t d = (s_out[static_cast<size_t>(p) * W + comp] >> shift) & 255u;
                out[static_cast<size_t>(s_gdst[d] + p) * W + c] = s_out[q];
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// K3: head flags, decoupled look-back scan, map scatter, unique compaction.
struct UniqueArgs {
    const uint32_t* rows0;
    const uint32_t* rows1;
    const uint32_t* plan;
    uint64_t* desc;     // [ntiles]
    uint32_t* counter;  // tile-id counter
    const uint32_t* status;
    uint32_t* map;      // map[org_id] = new_idx
    uint32_t* out_vtx;  // [U][D]
    unsigned long long* count;
    uint32_t* sc_org;   // optional scratch outputs
    uint8_t* sc_nodup;
    uint32_t* sc_new;
    uint32_t* sc_perm;
    uint32_t n;
    uint32_t ntiles;
    int dim;
};

template <int W_CT, int IPT>
struct UniqueTraits {
    static constexpr int kTile = kBlock * IPT;
    static __host__ __device__ size_t smem_bytes(int W) {
        return static_cast<size_t>(kTile) * W * 4 + (64 + kWarps + 8) * 4 + 16;
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

    extern __shared__ __align__(128) uint32_t smem[];
    uint32_t* s_rows = smem;
    uint32_t* s_prev = s_rows + static_cast<size_t>(TILE) * W;  // up to 64 words
    uint32_t* s_warp = s_prev + 64;
    uint32_t* s_misc = s_warp + kWarps;
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_misc + 8);

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    if (tid == 0) {
        mbar_init(s_bar, 1);
        fence_mbar_init();
    }
    __syncthreads();

    for (uint32_t iter = 0;; ++iter) {
        if (tid == 0) s_misc[0] = atomicAdd(a.counter, 1u);
        __syncthreads();
        const uint32_t tile = s_misc[0];
        if (tile >= a.ntiles) break;
        const uint32_t base = tile * static_cast<uint32_t>(TILE);
        const uint32_t tile_n = min(static_cast<uint32_t>(TILE), a.n - base);
        if (tid == 0) stage_tile(s_rows, rows + static_cast<size_t>(base) * W, tile_n * W * 4u, s_bar);
        if (tile > 0 && tid < static_cast<uint32_t>(D)) s_prev[tid] = rows[static_cast<size_t>(base - 1) * W + tid];
        mbar_wait(s_bar, iter & 1u);
        __syncthreads();

        // ---- phase 1: head flags (warp-striped rows) and per-warp totals
        uint32_t bal[IPT];
        uint32_t wtotal = 0;
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
            bool head = false;
            if (p < tile_n) {
                if (base + p == 0u) {
                    head = true;
                } else {
                    const uint32_t* cur = s_rows + static_cast<size_t>(p) * W;
                    const uint32_t* prv = p ? cur - W : s_prev;
                    if constexpr (W_CT > 0) {
#pragma unroll
                        for (int c = 0; c < W_CT - 1; ++c) head |= cur[c] != prv[c];
                    } else {
                        for (int c = 0; c < D; ++c) head |= cur[c] != prv[c];
                    }
                }
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

        // ---- decoupled look-back over tiles (warp 0, 32 predecessors per step)
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
                    const uint64_t dd = t >= 0 ? wait_desc(a.desc + t, 1u) : pack_desc(1u, kPrefix, 0u);
                    const uint32_t pm = __ballot_sync(kFull, desc_flag(dd) == kPrefix);
                    if (pm) {
                        const uint32_t first = __ffs(pm) - 1;
                        excl += warp_sum(lane <= first ? desc_value(dd) : 0u);
                        break;
                    }
                    excl += warp_sum(desc_value(dd));
                    hi -= 32;
                }
                if (lane == 0) st_relaxed(mine, pack_desc(1u, kPrefix, excl + ttotal));
            }
            if (lane == 0) s_misc[1] = excl;
        }
        __syncthreads();
        const uint32_t tprefix = s_misc[1];
        if (tid == 0 && tile == a.ntiles - 1) *a.count = static_cast<unsigned long long>(tprefix) + ttotal;

        // ---- phase 2: new index per slot, map scatter, unique rows out
        uint32_t running = tprefix + wexcl;
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
            if (p < tile_n) {
                const uint32_t* row = s_rows + static_cast<size_t>(p) * W;
                const uint32_t nidx = running + __popc(bal[r] & lanemask_le()) - 1u;
                const uint32_t org = row[D];
                a.map[org] = nidx;
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
