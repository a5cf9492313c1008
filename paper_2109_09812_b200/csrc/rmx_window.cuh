// rmx_window.cuh -- window mode: packed u32 keys sorted by their top 16 bits only, the low 16
// bits resolved by a presence bitmap per window (plan packed-section word 6).
//
// The reference's order is the key order and a key's new index is the number of distinct keys
// below it (pipeline.py:72-113).  For u32 packed keys of 25..32 bits (four 8-bit LSD passes) the
// packed path runs passes 2 and 3 only: the rows come out grouped by "window" = key >> 16, in
// window order.  Per window one CTA marks the low 16 bits of its rows in a 2^16-bit shared-memory
// bitmap, takes per-word prefix popcounts, learns the window's first new index from its
// predecessors (decoupled look-back over windows), and then
//   * writes the window's distinct keys in order (set bits, ascending) to ukeys for k_unpack_pk,
//   * gives every row its new index = base + set bits below its key, and writes (origin, new
//     index) pairs bucketed by origin for k_map_fill (as k_unique_pk does).
// Passes 0, 1, k_head_count_pk, k_tile_scan and k_unique_pk do not run.  The unused rows (no
// index reads their map entries, and the replacement row they stand for is a used row, so the
// distinct keys are those of the used rows) would all share the replacement key and form one giant
// window: without soup mode the first window pass drops them (pk[5]); in soup mode they stay, with
// keys spread by k_pack (a used neighbour's key or a row hash), and this kernel skips their
// origins >= I.  A window of more than kWinMaxRows rows (keys whose top 16 bits barely vary)
// would serialise on one CTA: k_win_bounds then sets the fallback word (pk[7]) and the full packed
// path runs after all (the digit byte 0 re-extracted, four passes over the window-grouped rows,
// the usual unique kernels).  Window mode is decided on the device (k_win_decide) for D <= 3 and
// no scratch request; RMX_WINDOW=0 turns it off.
#pragma once

#include "rmx_packed.cuh"

namespace rmx {

constexpr uint32_t kWinCount = 1u << 16;        // windows (key >> 16)
constexpr uint32_t kWinWords = (1u << 16) / 32;  // bitmap words per window
constexpr uint32_t kWinMaxRows = 1u << 21;      // larger windows take the fallback

__device__ __forceinline__ bool win_active(const uint32_t* plan, int D) {
    const uint32_t* pk = plan + pk_base(4 * D);
    return pk[0] == 1u && pk[6] != 0u && pk[7] == 0u;
}
__device__ __forceinline__ bool win_fallback(const uint32_t* plan, int D) {
    const uint32_t* pk = plan + pk_base(4 * D);
    return pk[0] == 1u && pk[6] != 0u && pk[7] != 0u;
}

// after the final plan (and the re-plan of a failed speculative plan: gate)
// (after the soup decision): soup mode keeps the unused rows (k_pack spreads their keys, the
// window kernel skips their origins >= I), else the first window pass drops them and counts the
// rows it keeps into *win_rows
__global__ void k_win_decide(uint32_t* plan, int D, int allow, const uint32_t* status, const uint32_t* gate,
                             const uint32_t* soup, uint32_t* win_rows, uint32_t n) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (threadIdx.x != 0 || *status) return;
    if (gate && !(*gate & 2u)) return;  // (kSpecMiss)
    uint32_t* pk = plan + pk_base(4 * D);
    const bool win = allow && pk[0] == 1u && pk[1] == 1u && pk[3] == 4u;
    const bool drop = win && !(soup && *soup);
    pk[5] = drop ? 1u : 0u;
    pk[6] = win ? 1u : 0u;
    pk[7] = 0u;
    *win_rows = drop ? 0u : n;
}

struct WinArgs {
    const uint32_t* plan;
    const uint32_t* keys;  // sorted by window (the final packed buffer)
    const uint32_t* vals;  // origins, same order
    uint2* pairs;          // bucketed (origin, new index) pairs (the other buffer)
    uint32_t* wstart;      // [kWinCount] first row of every window, 0xFFFFFFFF = empty
    uint32_t* wend;        // [kWinCount] one past its last row
    uint64_t* desc;        // [kWinCount] look-back descriptors
    uint32_t* counter;     // window counter
    uint32_t* fill;        // [256] pair bucket fill counters
    uint32_t* ukeys;       // [U] packed key of every distinct key
    unsigned long long* count;
    uint32_t* plan_w;      // plan, for the fallback word
    const uint32_t* status;
    uint32_t n;            // rows: *win_rows (the used rows the window passes keep)
    int dim;
    int bucket_shift;
    const uint32_t* win_rows;
    uint32_t n_slots;       // vertex slots V (the row buffers' extent)
    const uint32_t* soup;   // soup mode: I; rows of origin >= I are unused (kept, not dropped)
};

// first row and one past the last row of every non-empty window (empty windows keep wstart =
// 0xFFFFFFFF; their wend is never read), eight rows per thread; and the fallback decision: rows
// p = j * kWinProbe and p + kWinProbe in one window mean a window of more than kWinProbe rows
// (every window of more than kWinMaxRows = 2 kWinProbe rows holds such a pair), which would
// serialise on one CTA -- the full packed path runs instead (pk[7])
constexpr uint32_t kWinProbe = kWinMaxRows / 2;
__global__ void __launch_bounds__(kBlock) k_win_bounds(WinArgs a) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (*a.status || !win_active(a.plan, a.dim)) return;
    const uint32_t n = *a.win_rows;
    const uint32_t groups = (n + 7u) / 8u;  // eight rows per thread: two 16-byte loads in flight
    const uint32_t stride = gridDim.x * kBlock;
    for (uint32_t g = blockIdx.x * kBlock + threadIdx.x; g < groups; g += stride) {
        const uint32_t p0 = 8u * g;
        uint32_t w[8];
        if (p0 + 7u < n) {
            const uint4 k0 = __ldcs(reinterpret_cast<const uint4*>(a.keys) + 2 * g);
            const uint4 k1 = __ldcs(reinterpret_cast<const uint4*>(a.keys) + 2 * g + 1);
            w[0] = k0.x >> 16;
            w[1] = k0.y >> 16;
            w[2] = k0.z >> 16;
            w[3] = k0.w >> 16;
            w[4] = k1.x >> 16;
            w[5] = k1.y >> 16;
            w[6] = k1.z >> 16;
            w[7] = k1.w >> 16;
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) w[j] = p0 + j < n ? __ldg(a.keys + p0 + j) >> 16 : 0xFFFFFFFFu;
        }
        // the previous row's window: the lane before's last row (lane 0 loads it)
        uint32_t prev = __shfl_up_sync(__activemask(), w[7], 1);
        if ((threadIdx.x & 31u) == 0u) prev = p0 ? __ldg(a.keys + p0 - 1u) >> 16 : 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t p = p0 + static_cast<uint32_t>(j);
            if (p >= n) break;
            if (w[j] != prev) {
                a.wstart[w[j]] = p;
                if (p) a.wend[prev] = p;
            }
            if (p + 1u == n) a.wend[w[j]] = n;
            prev = w[j];
        }
        if (p0 % kWinProbe == 0u && p0 + kWinProbe < n && (__ldg(a.keys + p0 + kWinProbe) >> 16) == w[0])
            a.plan_w[pk_base(4 * a.dim) + 7] = 1u;  // the full packed path runs instead
    }
}

// The window's first new index: decoupled look-back over the windows before it (warp 0; the
// window's aggregate was published earlier).  Returns the exclusive prefix and publishes the
// inclusive one.
__device__ __forceinline__ uint32_t win_lookback(const WinArgs& a, uint32_t w, uint32_t total) {
    const uint32_t lane = threadIdx.x & 31u;
    uint64_t* mine = a.desc + w;
    uint32_t excl = 0;
    if (w == 0) return 0u;
    int64_t hi = static_cast<int64_t>(w) - 1;
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
    if (lane == 0) st_relaxed(mine, pack_desc(1u, kPrefix, excl + total));
    return excl;
}

// A row's slot in its origin bucket is warp-aggregated (bucket_slot, rmx_common.cuh: rows of a
// window sit in origin order, so a warp's rows often share a bucket); the marks and bucket counts
// stay plain fire-and-forget atomics (MATCH.ANY aggregation of those measured slower on C2 / C3).

// Rows are staged in shared memory by bulk copies (keys + origins).  A window of up to kWinCap rows
// is one chunk; a larger one is processed in chunks of kWinCap rows (marked chunk by chunk, then
// re-staged for the pairs).  3 CTAs per SM.
constexpr uint32_t kWinCap = 6656;
constexpr uint32_t kWinStage = kWinCap + 8;  // + 16-byte alignment slack
// 3 CTAs of 256 threads per SM (measured: 2 x 512 threads, 1.68 vs 1.42 ms on C2)
constexpr int kWinThreads = 256, kWinWarps = kWinThreads / 32, kWinMinBlocks = 3;
static_assert(kWinThreads >= 256, "one thread per origin bucket");
struct WinSmem {
    static constexpr size_t kKey = 0, kVal = kWinStage, kBm = 2 * kWinStage, kPre = kBm + kWinWords,
                            kBcnt = kPre + kWinWords, kBcur = kBcnt + 256, kBglob = kBcur + 256,
                            kWarp = kBglob + 256, kMisc = kWarp + 2 * kWinWarps, kBar = kMisc + 8, kWordsTotal = kBar + 2;
    static __host__ __device__ size_t bytes() { return kWordsTotal * 4; }
};

__global__ void __launch_bounds__(kWinThreads, kWinMinBlocks) k_win_unique(WinArgs a) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (*a.status || !win_active(a.plan, a.dim)) return;
    a.n = *a.win_rows;
    uint32_t* sm = dyn_smem<uint32_t>();
    uint32_t* s_key = sm + WinSmem::kKey;  // staged keys, then the local new index of every row
    uint32_t* s_val = sm + WinSmem::kVal;  // staged origins
    uint32_t* s_bm = sm + WinSmem::kBm;
    uint32_t* s_pre = sm + WinSmem::kPre;
    uint32_t* s_bcnt = sm + WinSmem::kBcnt;
    uint32_t* s_bcur = sm + WinSmem::kBcur;
    uint32_t* s_bglob = sm + WinSmem::kBglob;
    uint32_t* s_warp = sm + WinSmem::kWarp;
    uint32_t* s_misc = sm + WinSmem::kMisc;
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(sm + WinSmem::kBar);
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const int bs = a.bucket_shift;
    constexpr uint32_t kWpt = kWinWords / kWinThreads;  // bitmap words per thread
    // soup mode keeps the unused rows (origins >= I): they are skipped here
    const uint32_t lim = a.plan[pk_base(4 * a.dim) + 5] == 0u && a.soup ? *a.soup : 0xFFFFFFFFu;
    if (tid == 0) {
        mbar_init(s_bar, 1);
        fence_mbar_init();
    }
    uint32_t phase = 0;
    // rows [cs, cs + cr) to s_key / s_val from offset (cs & 3) on (the 16-byte aligned superset;
    // the row buffers extend past V to a multiple of 4 rows); all threads call it
    auto stage = [&](uint32_t cs, uint32_t cr) -> uint32_t {
        const uint32_t s4 = cs & ~3u, e4 = (cs + cr + 3u) & ~3u;
        __syncthreads();  // the previous chunk's readers are done
        if (tid == 0) stage_tile2(s_key, a.keys + s4, (e4 - s4) * 4u, s_val, a.vals + s4, (e4 - s4) * 4u, s_bar);
        mbar_wait(s_bar, phase);
        phase ^= 1u;
        return cs - s4;
    };
    for (uint32_t it = 0;; ++it) {
        uint32_t* slot = s_misc + (it & 1u) * 2;  // [0] window, [1] its base (alternating slots)
        if (tid == 0) slot[0] = atomicAdd(a.counter, 1u);
        __syncthreads();
        const uint32_t w = slot[0];
        if (w >= kWinCount) break;
        const uint32_t s = a.wstart[w];
        const uint32_t rows = s == 0xFFFFFFFFu ? 0u : a.wend[w] - s;
        if (rows == 0u) {  // empty: aggregate 0 (the last window resolves the count)
            if (w == kWinCount - 1) {
                if (warp == 0) {
                    if (lane == 0) st_relaxed(a.desc + w, pack_desc(1u, kAggregate, 0u));
                    const uint32_t excl = win_lookback(a, w, 0u);
                    if (lane == 0) *a.count = excl;
                }
            } else if (tid == 0) {
                st_relaxed(a.desc + w, pack_desc(1u, w == 0 ? kPrefix : kAggregate, 0u));
            }
            continue;
        }
        const bool one = rows <= kWinCap;
        constexpr uint32_t csz = kWinCap;
        const uint32_t nch = (rows + csz - 1u) / csz;
#pragma unroll
        for (uint32_t j = 0; j < kWpt; ++j) s_bm[tid * kWpt + j] = 0u;
        if (tid < 256u) s_bcnt[tid] = 0u;
        // ---- mark the low 16 bits, chunk by chunk (a one-chunk window also counts its buckets)
        uint32_t off = 0;
        for (uint32_t ch = 0; ch < nch; ++ch) {
            const uint32_t cr = min(csz, rows - ch * csz);
            off = stage(s + ch * csz, cr);
            for (uint32_t q = tid; q < cr; q += kWinThreads) {
                const uint32_t k = s_key[off + q] & 0xFFFFu;
                const uint32_t org = s_val[off + q];
                if (org < lim) {
                    atomicOr(s_bm + (k >> 5), 1u << (k & 31u));
                    if (one) atomicAdd(s_bcnt + (org >> bs), 1u);
                }
            }
        }
        __syncthreads();
        // ---- per-word prefix popcounts, the window's distinct keys; publish the aggregate (a
        // one-chunk window scans its bucket counts in the same block scan: counts < 2^16 each)
        uint32_t wb[kWpt], cnt = 0;
#pragma unroll
        for (uint32_t j = 0; j < kWpt; ++j) {
            wb[j] = s_bm[tid * kWpt + j];
            cnt += __popc(wb[j]);
        }
        const uint32_t bc1 = one && tid < 256u ? s_bcnt[tid] : 0u;
        uint32_t both;
        const uint32_t run2 = block_exclusive_scan<kWinWarps>(cnt | (bc1 << 17), s_warp, both);
        const uint32_t total = both & 0x1FFFFu;  // (distinct keys <= 2^16 in bits 0..16, rows < 2^15 above)
        uint32_t run = run2 & 0x1FFFFu;
        const uint32_t pre0 = run;  // distinct keys before this thread's bitmap words
#pragma unroll
        for (uint32_t j = 0; j < kWpt; ++j) {
            s_pre[tid * kWpt + j] = run;
            run += __popc(wb[j]);
        }
        if (tid == 0) st_relaxed(a.desc + w, pack_desc(1u, w == 0 ? kPrefix : kAggregate, total));
        // ---- pairs, chunk by chunk (a one-chunk window is still staged)
        // bucket space from the combined scan: one global reservation per bucket (its round trip
        // overlaps the new-index pass below)
        const uint32_t bstart1 = run2 >> 17;
        uint32_t bfill1 = 0u;
        if (one && tid < 256u) {
            s_bcur[tid] = bstart1;
            if (bc1) bfill1 = atomicAdd(a.fill + tid, bc1);
        }
        for (uint32_t ch = 0; ch < nch; ++ch) {
            const uint32_t cr = min(csz, rows - ch * csz);
            if (!one) {
                off = stage(s + ch * csz, cr);
                if (tid < 256u) s_bcnt[tid] = 0u;
            }
            __syncthreads();  // (s_pre, s_bcnt, s_bcur, s_bglob)
            // local new index of every row (in place; a chunk of a larger window also counts its
            // buckets); warp 0 then looks back
#pragma unroll 4
            for (uint32_t q = tid; q < cr; q += kWinThreads) {
                if (s_val[off + q] < lim) {
                    const uint32_t k = s_key[off + q] & 0xFFFFu;
                    const uint32_t wd = k >> 5;
                    s_key[off + q] = s_pre[wd] + __popc(s_bm[wd] & ((1u << (k & 31u)) - 1u));
                    if (!one) atomicAdd(s_bcnt + (s_val[off + q] >> bs), 1u);
                }
            }
            if (ch == 0 && warp == 0) {
                const uint32_t excl = win_lookback(a, w, total);
                if (lane == 0) slot[1] = excl;
            }
            if (one && bc1) s_bglob[tid] = (tid << bs) + bfill1 - bstart1;
            __syncthreads();
            if (!one) {  // bucket space: a block scan, one global reservation per bucket
                const uint32_t bc = tid < 256u ? s_bcnt[tid] : 0u;
                uint32_t chunk_rows;
                const uint32_t bstart = block_exclusive_scan<kWinWarps>(bc, s_warp + kWinWarps, chunk_rows);
                if (tid < 256u) s_bcur[tid] = bstart;
                if (bc) s_bglob[tid] = (tid << bs) + atomicAdd(a.fill + tid, bc) - bstart;
                __syncthreads();
            }
            const uint32_t base = slot[1];
            // every used row's (origin, new index) pair straight to its slot in its bucket's run
            // (warp-aggregated slots; the run's stores merge in L2 -- measured faster than a
            // shared-memory permutation and a coalesced copy-out: 1.34 vs 1.42 ms on C2)
#pragma unroll 2
            for (uint32_t q0 = 0; q0 < cr; q0 += kWinThreads) {  // (warp-uniform)
                const uint32_t q = q0 + tid;
                const uint32_t org = q < cr ? s_val[off + q] : 0xFFFFFFFFu;
                const bool valid = org < lim;
                const uint32_t pos = bucket_slot(s_bcur, valid, org >> bs);
                if (valid) {
                    RMX_CHECK_INDEX(s_bglob[org >> bs] + pos, a.n_slots);
                    a.pairs[s_bglob[org >> bs] + pos] = make_uint2(org, base + s_key[off + q]);
                }
            }
        }
        // ---- the window's distinct keys out, ascending
        const uint32_t base = slot[1];
        if (tid == 0 && w == kWinCount - 1) *a.count = static_cast<unsigned long long>(base) + total;
        {
            uint32_t r = base + pre0;
#pragma unroll
            for (uint32_t j = 0; j < kWpt; ++j) {
                uint32_t m = wb[j];
                while (m) {
                    const uint32_t b = __ffs(m) - 1u;
                    RMX_CHECK_INDEX(r, a.n);
                    a.ukeys[r++] = (w << 16) | ((tid * kWpt + j) << 5) | b;
                    m &= m - 1u;
                }
            }
        }
        __syncthreads();  // the staging area and the bitmap are reused
    }
}

// fallback: the digit byte 0 of the window-grouped rows for the full packed passes; in soup mode
// the unused rows (origins >= I) first get the replacement row's key back (k_pack spread their
// keys for the windows; the full path counts every row's key)
__global__ void __launch_bounds__(kBlock) k_win_digit0(const uint32_t* plan, int D, uint32_t* keys, const uint32_t* vals,
                                                       uint8_t* digits, const uint32_t* win_rows, const uint32_t* soup,
                                                       const uint32_t* status) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (*status || !win_fallback(plan, D)) return;
    const uint32_t n = win_rows[0];
    const uint32_t lim = plan[pk_base(4 * D) + 5] == 0u && soup ? *soup : 0xFFFFFFFFu;
    const uint32_t repl = win_rows[1];
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    for (uint64_t p = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x; p < n; p += stride) {
        uint32_t k = keys[p];
        if (__ldg(vals + p) >= lim) keys[p] = k = repl;
        digits[p] = static_cast<uint8_t>(k);
    }
}

}  // namespace rmx
