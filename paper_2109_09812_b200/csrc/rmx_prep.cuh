// rmx_prep.cuh -- K1 mark, K1b row build, plan, first-pass histogram (AoS row path).
#pragma once

#include "rmx_base.cuh"

namespace rmx {

// ---------------------------------------------------------------------------
// K1: mark used vertices; any index >= n_vtx sets the status bit.
// Each warp looks at its first 128 indices: when they fall in a window of
// kMarkWindow vertices (soups, grid meshes: indices in or near element order)
// it writes the byte flags directly -- the window's sectors merge in L2.
// Otherwise (shuffled indexed meshes) it sets bits in a bit set instead (V/8
// bytes, L2-resident up to ~10^9 vertices) with atomicOr: a direct byte store
// there costs a DRAM read-modify-write per index.  Either choice is correct
// for any index order.  k_expand_marks ORs the bit set into the byte flags.
constexpr uint32_t kMarkWindow = 1u << 16;

struct MarkArgs {
    const uint32_t* idx;
    uint64_t n_idx;
    uint64_t n_vtx;
    uint8_t* flags;   // [n_vtx] zeroed
    uint32_t* bits;   // [ceil(n_vtx / 32)] zeroed
    uint32_t* status;
    int vec;          // idx 16-byte aligned
    uint32_t* order;  // bit 0 set: the indices are not strictly increasing (soup mode, rmx_packed.cuh)
};

__global__ void __launch_bounds__(kBlock) k_mark(MarkArgs a) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const uint64_t gtid = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31u;
    bool bad = false, unordered = false;  // unordered: some idx[i] >= idx[i + 1]
    uint64_t done = 0;
    if (a.vec) {
        const uint64_t n4 = a.n_idx >> 2;
        const uint4* i4 = reinterpret_cast<const uint4*>(a.idx);
        const uint64_t wbase = gtid - lane;  // warp-uniform trip count for the vote below
        int local = -1;                      // decided on the warp's first group of indices
        for (uint64_t i0 = wbase; i0 < n4; i0 += stride) {
            const uint64_t i = i0 + lane;
            uint32_t x[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
            if (i < n4) {
                const uint4 v = __ldcs(i4 + i);
                x[0] = v.x;
                x[1] = v.y;
                x[2] = v.z;
                x[3] = v.w;
            }
            // order: within the group, and against the next group's first index (the next lane's,
            // or a load when the next group is another warp's or the scalar tail's)
            uint32_t nx = __shfl_down_sync(kFull, x[0], 1);
            if ((lane == 31u || i + 1 >= n4) && 4 * (i + 1) < a.n_idx) nx = __ldg(a.idx + 4 * (i + 1));
            if (i < n4)
                unordered = unordered || !(x[0] < x[1] && x[1] < x[2] && x[2] < x[3] &&
                                           (4 * (i + 1) >= a.n_idx || x[3] < nx));
            uint32_t lo = 0xFFFFFFFFu, hi = 0u;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (x[k] < a.n_vtx) {
                    lo = min(lo, x[k]);
                    hi = max(hi, x[k]);
                } else if (i < n4) {
                    bad = true;
                }
            }
            if (local < 0) {
                const uint32_t wlo = __reduce_min_sync(kFull, lo), whi = __reduce_max_sync(kFull, hi);
                local = (wlo == 0xFFFFFFFFu || whi - wlo < kMarkWindow) ? 1 : 0;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (x[k] < a.n_vtx) {
                    if (local) a.flags[x[k]] = 1;
                    else atomicOr(a.bits + (x[k] >> 5), 1u << (x[k] & 31u));
                }
            }
        }
        done = n4 << 2;
    }
    for (uint64_t i = done + gtid; i < a.n_idx; i += stride) {
        const uint32_t x = __ldcs(a.idx + i);
        if (x < a.n_vtx) a.flags[x] = 1;
        else bad = true;
        if (i + 1 < a.n_idx && !(x < __ldg(a.idx + i + 1))) unordered = true;
    }
    if (__any_sync(kFull, bad) && lane == 0u) atomicOr(a.status, RMX_STATUS_INDEX_OUT_OF_RANGE);
    if (__any_sync(kFull, unordered) && lane == 0u && a.order) atomicOr(a.order, 1u);
}

// flags |= bit set (one word of 32 vertices per thread; words with no bit
// set -- all of them when no warp took the scattered path -- cost one load).
__global__ void __launch_bounds__(kBlock) k_expand_marks(const uint32_t* bits, uint64_t n_vtx, uint8_t* flags) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const uint64_t nw = (n_vtx + 31) >> 5;
    for (uint64_t w = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x; w < nw; w += stride) {
        uint32_t b = __ldcs(bits + w);
        while (b) {
            const uint32_t t = __ffs(b) - 1u;
            flags[(w << 5) + t] = 1;
            b &= b - 1u;
        }
    }
}

// ---------------------------------------------------------------------------
// K1b (AoS mode): cleaned (key words, origin) rows and the digit histograms
// of component D-1 (passes 0..3: the first executed pass is almost always
// among them).
struct BuildArgs {
    const uint32_t* vtx;
    const uint8_t* flags;
    const uint32_t* idx;  // idx[0] is the replacement vertex (pipeline.py:148)
    uint32_t* rows;
    uint32_t* hist;       // [4D][256]; this kernel fills passes 0..3
    const uint32_t* plan;
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
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    const int D = D_CT > 0 ? D_CT : a.dim;
    const int W = D + 1;
    __shared__ uint32_t s_hist[4 * 256];
    for (int i = threadIdx.x; i < 4 * 256; i += kBlock) s_hist[i] = 0u;
    __syncthreads();
    if (*a.status || a.plan[pk_base(4 * D)] != 0u) return;  // uniform; packed mode builds no rows

    const uint32_t r0 = a.idx[0];
    const uint32_t* repl = a.vtx + static_cast<size_t>(r0) * D;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const uint64_t start = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    uint32_t rl[4] = {0u, 0u, 0u, 0u};

    if constexpr (D_CT > 0) {
        uint32_t ref[D_CT];
#pragma unroll
        for (int c = 0; c < D_CT; ++c) ref[c] = __ldg(repl + c);
        auto emit = [&](uint64_t i, uint32_t (&k)[D_CT]) {
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
    } else {
        for (uint64_t i = start; i < a.n; i += stride) {
            const bool used = a.flags[i] != 0;
            const uint32_t* srow = used ? a.vtx + i * D : repl;
            uint32_t* dst = a.rows + i * W;
            for (int c = 0; c < D; ++c) {
                const uint32_t k = __ldg(srow + c);
                dst[c] = k;
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
}

// ---------------------------------------------------------------------------
// plan (one thread): from the per-component varying-bit masks decide between
//  * packed mode -- at most 64 varying bits in at most kMaxRuns runs: the
//    key is compacted to a u32/u64 and sorted in ceil(B/8) passes; and
//  * AoS mode -- a byte pass executes iff its digit is not constant over all
//    keys; passes chain to the next executed one, buffers ping-pong.
// allow_hash: when the key does not pack into 64 bits, take hash mode (rmx_hash.cuh) instead of
// sorting the whole vertex set as AoS rows; the AoS pass schedule is made either way (hash mode
// sorts its candidate rows with it).
__device__ void plan_body(const uint32_t* vary, const uint32_t* fields, uint32_t* plan, int D, bool allow_hash) {
    const int P = 4 * D;
    uint32_t* pk = plan + pk_base(P);
    uint32_t* rk = plan + pk_rank_base(P);
    uint32_t* vb = plan + pk_value_base(P);
    vb[0] = 0u;
    vb[1] = 0u;
    pk[5] = 0u;  // window mode (rmx_window.cuh k_win_decide): drop, on, fallback
    pk[6] = 0u;
    pk[7] = 0u;
    uint32_t bits = 0, runs = 0, cand = 0;
    bool fits = true;
    for (int c = D - 1; c >= 0 && fits; --c) {
        const uint32_t c_lo = bits;
        uint32_t m = vary[c];
        // field rank (see rmx_base.cuh) when it needs fewer bits than the varying field bits
        uint32_t rank_bits = 0;
        bool ranked = false;
        if (D <= kMaxRankDim) {
            uint32_t distinct = 0;
            for (int w = 0; w < kFieldWords; ++w) distinct += __popc(fields[c * kFieldWords + w]);
            while ((1u << rank_bits) < distinct) ++rank_bits;
            ranked = rank_bits < static_cast<uint32_t>(__popc(m >> kFieldLo));
        }
        rk[c] = 0u;
        if (ranked) m &= (1u << kFieldLo) - 1u;
        while (m) {
            const uint32_t lo = __ffs(m) - 1u;
            const uint32_t len = __ffs(~(m >> lo)) ? __ffs(~(m >> lo)) - 1u : 32u - lo;
            if (runs == static_cast<uint32_t>(kMaxRuns) || bits + len > 64u) {
                fits = false;
                break;
            }
            pk[8 + 4 * runs + 0] = static_cast<uint32_t>(c);
            pk[8 + 4 * runs + 1] = lo;
            pk[8 + 4 * runs + 2] = len;
            pk[8 + 4 * runs + 3] = bits;
            ++runs;
            bits += len;
            m = len >= 32u ? 0u : (m & ~(((1u << len) - 1u) << lo));
        }
        if (ranked && fits) {
            if (bits + rank_bits > 64u) {
                fits = false;
            } else {
                rk[c] = (1u << 31) | (rank_bits << 16) | bits;
                bits += rank_bits;
            }
        }
        if (fits && D <= kMaxRankDim) {  // component c occupies key bits [c_lo, bits)
            const uint32_t w = bits - c_lo;
            uint32_t* e = vb + 4 + 4 * c;
            e[0] = c_lo;
            e[1] = w;
            e[2] = c_lo;
            e[3] = w;
            if (w >= static_cast<uint32_t>(kMinValueBits) && w <= static_cast<uint32_t>(kMaxValueBits)) cand |= 1u << c;
        }
    }
    if (fits) {
        for (;;) {  // the value-set byte maps must fit one CTA: drop the widest candidates
            uint32_t need = 0, widest = 0, wmax = 0;
            for (int c = 0; c < D && c < kMaxRankDim; ++c) {
                if (!((cand >> c) & 1u)) continue;
                const uint32_t w = vb[4 + 4 * c + 1];
                need += 1u << w;
                if (w > wmax) {
                    wmax = w;
                    widest = static_cast<uint32_t>(c);
                }
            }
            if (need <= kValueSetBytes) break;
            cand &= ~(1u << widest);
        }
        vb[1] = cand;
        const uint32_t npass = (bits + 7u) / 8u;
        pk[0] = 1u;
        pk[1] = bits > 32u ? 2u : 1u;
        pk[2] = bits;
        pk[3] = npass;
        pk[4] = runs;
        for (int p = 0; p < P; ++p) {
            plan[4 + p] = 0u;
            plan[4 + P + p] = 0u;
            plan[4 + 2 * P + p] = static_cast<uint32_t>(P);
        }
        plan[0] = npass & 1u;  // packed buffers ping-pong starting from buffer 0
        plan[1] = npass;
        plan[2] = 0u;
        plan[3] = 0u;
        return;
    }
    pk[0] = 0u;
    // AoS mode builds the rows in buffer 0; hash mode sorts its candidate rows from the buffer the
    // grouped rows are not in
    uint32_t cur = (allow_hash && !(kHashPasses & 1)) ? 1u : 0u, executed = 0, first = static_cast<uint32_t>(P),
             prev = static_cast<uint32_t>(P);
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
    plan[3] = (first < static_cast<uint32_t>(P) && first >= 4u) ? 1u : 0u;  // histogram not made by K1b / k_hash_dedup
    if (allow_hash) {  // rows grouped by hash, deduplicated per tile, the candidates sorted as AoS rows
        pk[0] = 2u;
        pk[1] = 0u;
        pk[2] = 0u;
        pk[3] = 0u;  // no packed passes
        pk[4] = 0u;
    }
}

__global__ void k_plan(const uint32_t* vary, const uint32_t* fields, uint32_t* plan, int D, const uint32_t* status,
                       int allow_hash, const uint32_t* gate = nullptr) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (*status || threadIdx.x != 0) return;
    if (gate && !(*gate & 2u)) return;  // the fallback of a failed speculative plan (kSpecMiss)
    plan_body(vary, fields, plan, D, allow_hash != 0);
}

// Histogram of the first executed pass when it lies outside component D-1
// (only then; exits immediately otherwise).
struct HistArgs {
    const uint32_t* rows;    // buffer 0; the rows of the first executed pass are in rows_alt when its
    const uint32_t* rows_alt;  // source parity says so (hash mode)
    uint32_t* hist;
    const uint32_t* plan;
    const uint32_t* status;
    uint32_t n;
    int dim;
    const uint32_t* n_cand;  // hash mode: the rows are the n_cand candidate rows
};

__global__ void __launch_bounds__(kBlock) k_first_hist(HistArgs a) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    const uint32_t mode = a.plan[pk_base(4 * a.dim)];
    if (*a.status || a.plan[3] == 0u || mode == 1u) return;
    const uint32_t n = mode == 2u ? *a.n_cand : a.n;
    const int Pd = 4 * a.dim;
    const uint32_t* rows = a.plan[4 + Pd + a.plan[2]] ? a.rows_alt : a.rows;
    __shared__ uint32_t s_h[256];
    s_h[threadIdx.x] = 0u;
    __syncthreads();
    const uint32_t p = a.plan[2];
    const int comp = a.dim - 1 - static_cast<int>(p >> 2);
    const int shift = 8 * static_cast<int>(p & 3u);
    const int W = a.dim + 1;
    uint32_t rl = 0u;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * kBlock)
        rl_push(rl, (__ldcs(rows + i * W + comp) >> shift) & 255u, s_h);
    if ((rl >> 8) != 0u) atomicAdd(s_h + (rl & 255u), rl >> 8);
    __syncthreads();
    if (s_h[threadIdx.x]) atomicAdd(a.hist + p * 256 + threadIdx.x, s_h[threadIdx.x]);
}

}  // namespace rmx
