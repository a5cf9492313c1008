// rmx_common.cuh -- sm_100a device helpers shared by the re-indexing kernels:
// warp intrinsics, relaxed GPU-scope atomics for decoupled look-back,
// mbarrier + cp.async.bulk (TMA bulk copy) tile staging.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rmx {

constexpr uint32_t kFull = 0xFFFFFFFFu;

// The one dynamic shared-memory declaration of the library: every kernel takes
// its dynamic shared memory from here (declarations with different alignments
// of the same extern array in one translation unit are ill-formed).
extern __shared__ __align__(128) unsigned char rmx_dyn_smem[];
template <typename T>
__device__ __forceinline__ T* dyn_smem() {
    return reinterpret_cast<T*>(rmx_dyn_smem);
}

// Checked build (-DRMX_CHECKED, tools/checked_probe.py): every scattered store of the pipeline
// counts an index past its array here (read by rmx_debug_oob_count); compiled out otherwise.
// It stands in for compute-sanitizer, which this GPU pool does not run.
#ifdef RMX_CHECKED
__device__ unsigned long long g_rmx_oob;
#define RMX_CHECK_INDEX(i, n)                                                              \
    do {                                                                                    \
        if (static_cast<unsigned long long>(i) >= static_cast<unsigned long long>(n))       \
            atomicAdd(&g_rmx_oob, 1ull);                                                    \
    } while (0)
#else
#define RMX_CHECK_INDEX(i, n) \
    do {                      \
    } while (0)
#endif

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint32_t lanemask_le() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
    return m;
}

// ---- GPU-scope relaxed accesses for look-back descriptors -----------------
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Look-back descriptor: [63:34] epoch, [33:32] flag, [31:0] value.
// The value is a count of rows, bounded by n_vertices < 2^32.
constexpr uint32_t kAggregate = 1u;
constexpr uint32_t kPrefix = 2u;

__device__ __forceinline__ uint64_t pack_desc(uint32_t epoch, uint32_t flag, uint32_t value) {
    return (static_cast<uint64_t>(epoch) << 34) | (static_cast<uint64_t>(flag) << 32) | value;
}
__device__ __forceinline__ uint32_t desc_epoch(uint64_t d) { return static_cast<uint32_t>(d >> 34); }
__device__ __forceinline__ uint32_t desc_flag(uint64_t d) { return static_cast<uint32_t>(d >> 32) & 3u; }
__device__ __forceinline__ uint32_t desc_value(uint64_t d) { return static_cast<uint32_t>(d); }

// Spin until the descriptor carries this epoch and a non-empty flag.
__device__ __forceinline__ uint64_t wait_desc(const uint64_t* p, uint32_t epoch) {
    uint64_t d = ld_relaxed(p);
    while (desc_epoch(d) != epoch || desc_flag(d) == 0u) {
        __nanosleep(32);
        d = ld_relaxed(p);
    }
    return d;
}

// ---- mbarrier + bulk async copy (TMA, non-tensor) --------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Order this thread's earlier generic-proxy shared-memory accesses (made
// visible to it by a preceding __syncthreads) before later async-proxy writes.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

// Global -> shared bulk copy completing `bytes` of transaction on `bar`.
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "RMX_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra RMX_WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// Stage `bytes` (rounded up to 16) from global `src` into shared `dst`.
// Called by one thread; everybody then waits on `bar` with `parity`.
__device__ __forceinline__ void stage_tile(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    const uint32_t b16 = (bytes + 15u) & ~15u;
    fence_proxy_async_smem();
    mbar_expect_tx(bar, b16);
    // one bulk op per 32 KiB keeps each request modest and lets the copy
    // engine pipeline the pieces
    constexpr uint32_t kChunk = 32768u;
    const char* s = static_cast<const char*>(src);
    char* d = static_cast<char*>(dst);
    for (uint32_t off = 0; off < b16; off += kChunk) {
        const uint32_t n = (b16 - off) < kChunk ? (b16 - off) : kChunk;
        bulk_g2s(d + off, s + off, n, bar);
    }
}

// Two ranges staged onto one barrier (keys + values of a packed tile).
__device__ __forceinline__ void stage_tile2(void* dst0, const void* src0, uint32_t bytes0, void* dst1, const void* src1,
                                            uint32_t bytes1, uint64_t* bar) {
    const uint32_t b0 = (bytes0 + 15u) & ~15u, b1 = (bytes1 + 15u) & ~15u;
    fence_proxy_async_smem();
    mbar_expect_tx(bar, b0 + b1);
    constexpr uint32_t kChunk = 32768u;
    for (uint32_t off = 0; off < b0; off += kChunk)
        bulk_g2s(static_cast<char*>(dst0) + off, static_cast<const char*>(src0) + off, min(kChunk, b0 - off), bar);
    for (uint32_t off = 0; off < b1; off += kChunk)
        bulk_g2s(static_cast<char*>(dst1) + off, static_cast<const char*>(src1) + off, min(kChunk, b1 - off), bar);
}

// The slot of this lane's row in bucket b (s_bcur: the buckets' next free slots), warp-aggregated:
// rows of a warp often share a bucket, and same-address shared atomics that return a value
// serialise.  All lanes call it (`valid` masks the rows).
__device__ __forceinline__ uint32_t bucket_slot(uint32_t* s_bcur, bool valid, uint32_t b) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t peers = __match_any_sync(kFull, valid ? b : 0xFFFFFFFFu);
    const uint32_t leader = __ffs(peers) - 1u;
    uint32_t pos = 0;
    if (valid && lane == leader) pos = atomicAdd(s_bcur + b, __popc(peers));
    return __shfl_sync(kFull, pos, leader) + __popc(peers & ((1u << lane) - 1u));
}

// ---- block scan over one value per thread ----------------------------------
// Exclusive scan of `v` across a block of NW warps; `s_warp` holds NW words and
// must not be reused until a later __syncthreads.
template <int NW>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp, uint32_t& total) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= static_cast<uint32_t>(o)) x += y;
    }
    if (lane == 31u) s_warp[warp] = x;
    __syncthreads();
    uint32_t before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const uint32_t t = s_warp[w];
        before += (static_cast<uint32_t>(w) < warp) ? t : 0u;
        all += t;
    }
    total = all;
    return before + x - v;
}

// Exclusive scan of counts[0, n) in place by one CTA of 1024 threads; returns
// the total.  Rounds of 8192 values (8 consecutive per thread), the next
// round's loads issued before this round's scan: one CTA is latency-bound, so
// the loads must be in flight together (a thread-serial walk over n / 1024
// values cost 47 us for 51K tile counts; this ~10 us).
__device__ __forceinline__ uint32_t block_scan_counts(uint32_t* counts, uint32_t n, uint32_t* s_warp) {
    constexpr uint32_t kPer = 8, kRound = 1024u * kPer;
    const uint32_t t = threadIdx.x;
    uint32_t cur[kPer], nxt[kPer];
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k) cur[k] = t * kPer + k < n ? counts[t * kPer + k] : 0u;
    uint32_t carry = 0;
    for (uint32_t base = 0; base < n; base += kRound) {
        const uint32_t nb = base + kRound;
#pragma unroll
        for (uint32_t k = 0; k < kPer; ++k) nxt[k] = nb + t * kPer + k < n ? counts[nb + t * kPer + k] : 0u;
        uint32_t sum = 0;
#pragma unroll
        for (uint32_t k = 0; k < kPer; ++k) sum += cur[k];
        uint32_t tot;
        uint32_t run = carry + block_exclusive_scan<32>(sum, s_warp, tot);
#pragma unroll
        for (uint32_t k = 0; k < kPer; ++k) {
            const uint32_t i = base + t * kPer + k;
            if (i < n) counts[i] = run;
            run += cur[k];
        }
        carry += tot;
        __syncthreads();  // s_warp is reused by the next round
#pragma unroll
        for (uint32_t k = 0; k < kPer; ++k) cur[k] = nxt[k];
    }
    return carry;
}

// Warp multi-split strategies (per pass, uniform):
//   kRankMatch  -- MATCH.ANY: ~2 SM-cycles per DISTINCT value in the warp on B200;
//   kRankBallot -- 8 bit-plane masks (redux.sync): ~21 SM-cycles per warp round regardless of entropy;
//   kRankAtomic -- OR lane bits into a per-warp smem mask per digit, read back.
// prefer: match when at most 16 digit bins are populated (from the global
// histogram, `h` = this thread's bin of a 256-thread block), ballot otherwise.
constexpr int kRankMatch = 0, kRankBallot = 1, kRankAtomic = 2;
__device__ __forceinline__ int choose_rank(uint32_t h, int forced) {
    const int populated = __syncthreads_count(h != 0u);
    if (forced >= 0) return forced;
    return populated <= 16 ? kRankMatch : kRankBallot;
}

// Stable warp ranking of IPT rounds of 8-bit digits (pk[r] = digit, 256 for
// rows past the end of a partial tile).  wh = this warp's 256 digit counters,
// wm = its 256 peer masks (kRankAtomic only); both zero on entry, wm zero on
// exit.  On return pk[r] = digit << 16 | rank among this warp's earlier rows
// with the same digit, and wh holds the warp's digit counts.  Peer masks of
// all rounds are formed first where possible (independent instructions);
// only the short counter read-modify-write chain is serial.
// peers &= { lanes whose (digit & mask) agrees with mine }
__device__ __forceinline__ void bit_plane_and(uint32_t& peers, uint32_t d, uint32_t mask) {
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t, bb, m;\n\t"
        "and.b32 t, %1, %2;\n\t"
        "setp.ne.u32 p, t, 0;\n\t"
        "vote.sync.ballot.b32 bb, p, 0xffffffff;\n\t"
        "selp.b32 m, 0, 0xffffffff, p;\n\t"
        "xor.b32 bb, bb, m;\n\t"
        "and.b32 %0, %0, bb;\n\t}"
        : "+r"(peers)
        : "r"(d), "r"(mask));
}

// Swizzled slot of digit d in a 256-entry per-warp counter table.  Digits of
// real keys are structured (float mantissas of lattice-like data keep their
// low bits constant while high bits vary), so the lanes of a warp touching
// distinct digits d = h*32 + c would all hit bank c; folding the high bits
// into the bank spreads them.  A bijection on [0, 256).
__device__ __forceinline__ uint32_t hsw(uint32_t d) { return d ^ (d >> 5); }

// Rank the IPT digits (pk[r] < 256, or 256 = invalid when PARTIAL) of this
// lane within the warp.  On return pk[r] = (hsw(d) << 16) | (rows of this warp
// with digit d before this one, counted on top of wh[hsw(d)]); wh[hsw(d)] has
// grown by the warp's count of digit d.
template <int IPT, bool PARTIAL = true>
__device__ __forceinline__ void warp_rank(uint32_t (&pk)[IPT], uint32_t* wh, uint32_t* wm, int mode, bool partial) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t bit = 1u << lane;
    const uint32_t lt = bit - 1u;
    uint32_t pm[IPT];
    if (mode == kRankMatch) {
#pragma unroll
        for (int r = 0; r < IPT; ++r) pm[r] = __match_any_sync(kFull, pk[r]);
    } else if (mode == kRankBallot) {
        // 8 bit planes; per bit one LOP3.P (test), VOTE, SEL and a 3-input LOP3
        // (peers &= ballot ^ ~mine): written in PTX so ptxas does not re-derive
        // the predicate or spill it into a register bitmask.
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t d = pk[r];
            uint32_t peers = kFull;
#pragma unroll
            for (int b = 0; b < 8; ++b) bit_plane_and(peers, d, 1u << b);
            pm[r] = peers;
        }
        if (PARTIAL && partial) {
#pragma unroll
            for (int r = 0; r < IPT; ++r) pm[r] &= __ballot_sync(kFull, pk[r] < 256u);
        }
    } else {
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t d = pk[r];
            const bool valid = !PARTIAL || d < 256u;
            const uint32_t ds = hsw(d & 255u);
            if (valid) atomicOr(wm + ds, bit);
            __syncwarp();
            pm[r] = valid ? wm[ds] : 0u;
            __syncwarp();
            if (valid && (pm[r] & lt) == 0u) wm[ds] = 0u;
            __syncwarp();
        }
    }
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
        const uint32_t d = pk[r];
        const uint32_t peers = pm[r];
        const bool valid = !PARTIAL || d < 256u;
        const uint32_t ds = hsw(d & 255u);
        const uint32_t before = valid ? wh[ds] : 0u;
        __syncwarp();
        if (valid && (peers & lt) == 0u) wh[ds] = before + __popc(peers);
        __syncwarp();
        pk[r] = (ds << 16) | (before + __popc(peers & lt));
    }
}

// Decoupled look-back for one digit column of the [tile][256] descriptor
// array: LB predecessors are read per round trip, and waiting on a
// not-yet-published descriptor backs off exponentially (spinning threads
// would otherwise steal issue slots from the CTAs doing real work).
#ifdef RMX_PHASES
__device__ unsigned long long g_lb_stats[4];  // windows, spins, look-backs, distance
#endif

template <int LB>
__device__ __forceinline__ uint32_t lookback_digit(const uint64_t* desc, uint32_t tile, uint32_t d, uint32_t epoch) {
    uint32_t excl = 0;
    int64_t t = static_cast<int64_t>(tile) - 1;
    uint32_t backoff = 32;
#ifdef RMX_PHASES
    uint32_t st_w = 0, st_s = 0;
#endif
    for (;;) {
#ifdef RMX_PHASES
        ++st_w;
#endif
        uint64_t v[LB];
#pragma unroll
        for (int j = 0; j < LB; ++j)
            v[j] = (t - j >= 0) ? ld_relaxed(desc + static_cast<size_t>(t - j) * 256 + d) : pack_desc(epoch, kPrefix, 0u);
        bool done = false;
#pragma unroll
        for (int j = 0; j < LB; ++j) {
            if (!done) {
                while (desc_epoch(v[j]) != epoch || desc_flag(v[j]) == 0u) {
#ifdef RMX_PHASES
                    ++st_s;
#endif
                    __nanosleep(backoff);
                    backoff = min(backoff * 2u, 1024u);
                    v[j] = ld_relaxed(desc + static_cast<size_t>(t - j) * 256 + d);
                }
                excl += desc_value(v[j]);
                done = desc_flag(v[j]) == kPrefix;
            }
        }
        if (done) {
#ifdef RMX_PHASES
            if (d == 0) {
                atomicAdd(g_lb_stats + 0, st_w);
                atomicAdd(g_lb_stats + 1, st_s);
                atomicAdd(g_lb_stats + 2, 1ull);
            }
#endif
            return excl;
        }
        t -= LB;
    }
}

// Programmatic dependent launch (the pipeline launches its kernels with
// cudaLaunchAttributeProgrammaticStreamSerialization): first thing in every
// pipeline kernel, before any global access, wait until the previous kernel of
// the stream has completed and its writes are visible.  The launch of this
// kernel then overlaps the previous kernel's drain instead of following its
// completion.  No explicit early trigger (griddepcontrol.launch_dependents):
// measured, CTAs parked in the wait while the previous grid's last wave runs
// cost more than they save on large grids (C2 7.46 -> 8.70 ms with it,
// 7.32 ms without; C1 0.48 -> 0.39 / 0.35 ms).  No-op without the attribute.
__device__ __forceinline__ void pdl_enter() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// L2 prefetch of the line holding p (streaming loops: the loads of a later
// iteration start while this one computes, without holding registers)
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

__device__ __forceinline__ uint32_t warp_sum(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

}  // namespace rmx
