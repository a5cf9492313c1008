// rmx_unique.cuh -- K3 head flags / look-back scan / compaction / bucketed pairs, K3b map fill, K4 remap (AoS row path).
#pragma once

#include "rmx_base.cuh"

namespace rmx {

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
    const uint32_t* n_cand;  // hash mode: the rows are the n_cand candidate rows
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
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    using T = UniqueTraits<W_CT, IPT>;
    constexpr int TILE = T::kTile;
    const int D = W_CT > 0 ? W_CT - 1 : a.dim;
    const int W = D + 1;
    const uint32_t mode = a.plan[pk_base(4 * D)];
    if (*a.status || mode == 1u) return;  // packed mode: k_unique_pk
    // AoS mode: the whole vertex set; hash mode: the n_cand candidate rows (their org is the group)
    const uint32_t n = mode == 2u ? *a.n_cand : a.n;
    const uint32_t ntiles = (n + static_cast<uint32_t>(TILE) - 1u) / static_cast<uint32_t>(TILE);
    const uint32_t* __restrict__ rows = a.plan[0] ? a.rows1 : a.rows0;
    uint2* __restrict__ pairs = reinterpret_cast<uint2*>(a.plan[0] ? const_cast<uint32_t*>(a.rows0)
                                                                    : const_cast<uint32_t*>(a.rows1));

    uint32_t* smem = dyn_smem<uint32_t>();
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
            if (t < ntiles) {
                const uint32_t tn = min(static_cast<uint32_t>(TILE), n - t * static_cast<uint32_t>(TILE));
                stage_tile(s_rows, rows + static_cast<size_t>(t) * TILE * W, tn * W * 4u, s_bar);
            }
        }
        s_bcnt[tid] = 0u;
        __syncthreads();
        const uint32_t tile = s_misc[0];
        if (tile >= ntiles) break;
        const uint32_t base = tile * static_cast<uint32_t>(TILE);
        const uint32_t tile_n = min(static_cast<uint32_t>(TILE), n - base);
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
        if (tid == 0 && tile == ntiles - 1) *a.count = static_cast<unsigned long long>(tprefix) + ttotal;

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
                    RMX_CHECK_INDEX(nidx, n);
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
            RMX_CHECK_INDEX(s_bglob[pr.x >> bs] + q, n);
            pairs[s_bglob[pr.x >> bs] + q] = pr;
        }
        __syncthreads();
    }
}

// K3b: map[org] = new_idx from the bucket-major pair array (streaming reads;
// the stores of concurrently running CTAs fall in one or two buckets, i.e. an
// L2-resident window of map, so partial sectors merge before write-back).
// mode_want 0: the final map -- from K3's pairs (packed / AoS modes) or from k_hash_pairs' pairs
// (hash mode: the other row buffer); one thread per two pairs (the many CTAs in flight keep the
// scattered stores of ~one bucket -- an L2-resident window of map -- going at once).
// mode_want 2: hash mode's rank_of[candidate] from the candidates' pairs; a grid-stride loop over a
// capped grid, so that the launch costs nothing in the other modes.
__global__ void __launch_bounds__(kBlock) k_map_fill(const uint32_t* plan, const uint32_t* rows0,
                                                      const uint32_t* rows1, uint32_t* map, uint32_t n,
                                                      const uint32_t* status, int dim, int mode_want,
                                                      const uint32_t* n_cand, const uint32_t* soup,
                                                      uint32_t* out_idx, const uint32_t* wfill, int bs) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (*status) return;
    const bool hash = plan[pk_base(4 * dim)] == 2u;
    // window mode (rmx_window.cuh): pairs for the used rows only -- bucket b holds wfill[b] pairs
    // from b << bs on (without soup mode's dense origins the buckets are not full)
    const bool win = mode_want == 0 && wfill && plan[pk_base(4 * dim)] == 1u && plan[pk_base(4 * dim) + 6] != 0u;
    auto live = [&](uint64_t p) {
        const uint32_t b = static_cast<uint32_t>(p >> bs);
        return !win || p - (static_cast<uint64_t>(b) << bs) < __ldg(wfill + b);
    };
    // soup mode (rmx_packed.cuh k_soup_decide): origins below I are index positions -- the map is
    // the output; origins >= I are unused rows, which no index reads
    const uint32_t n_used = (mode_want == 0 && soup) ? *soup : 0u;
    if (n_used) map = out_idx;
    const uint32_t lim = n_used ? n_used : 0xFFFFFFFFu;
    if (mode_want == 2) {
        if (!hash) return;
        n = *n_cand;
        const uint4* pairs = reinterpret_cast<const uint4*>(plan[0] ? rows0 : rows1);
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
        for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x; 2 * i < n; i += stride) {
            if (2 * i + 1 < n) {
                const uint4 v = __ldcs(pairs + i);
                RMX_CHECK_INDEX(v.x, n);
                RMX_CHECK_INDEX(v.z, n);
                map[v.x] = v.y;
                map[v.z] = v.w;
            } else {
                const uint2 v = reinterpret_cast<const uint2*>(pairs)[2 * i];
                RMX_CHECK_INDEX(v.x, n);
                map[v.x] = v.y;
            }
        }
        return;
    }
    const uint4* pairs = reinterpret_cast<const uint4*>((plan[0] != 0u) != hash ? rows0 : rows1);
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;  // two pairs per thread
    if (win) {
        for (uint64_t p = 2 * i; p < 2 * i + 2 && p < n; ++p)
            if (live(p)) {
                const uint2 v = reinterpret_cast<const uint2*>(pairs)[p];
                RMX_CHECK_INDEX(v.x, n);
                if (v.x < lim) map[v.x] = v.y;
            }
    } else if (2 * i + 1 < n) {
        const uint4 v = __ldcs(pairs + i);
        RMX_CHECK_INDEX(v.x, n);
        RMX_CHECK_INDEX(v.z, n);
        if (v.x < lim) map[v.x] = v.y;
        if (v.z < lim) map[v.z] = v.w;
    } else if (2 * i < n) {
        const uint2 v = reinterpret_cast<const uint2*>(pairs)[2 * i];
        RMX_CHECK_INDEX(v.x, n);
        if (v.x < lim) map[v.x] = v.y;
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
    const uint32_t* soup;  // soup mode: the map fill wrote the output indices already
};

__global__ void __launch_bounds__(kBlock) k_remap(RemapArgs a) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (*a.status || (a.soup && *a.soup)) return;
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

}  // namespace rmx
