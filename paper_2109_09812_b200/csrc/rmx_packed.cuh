// rmx_packed.cuh -- the packed-key path.
//
// Mesh coordinates rarely use all 32 bits of every component: lattice or
// quantised data leave exponent and low mantissa bits constant.  The plan
// (rmx_prep.cuh:k_plan) gathers the bits that vary over the cleaned vertex
// set into runs; when they total at most 64 bits the sort runs over
// (packed key, origin) pairs instead of full (D key words, origin) rows:
//
//   K1a  k_vary       OR over used rows of (key ^ replacement key), per component
//   K1b' k_pack       cleaned rows -> packed u32/u64 keys + origins (SoA), and the
//                     histogram of packed digit 0 (overwrite_unused pipeline.py:54-63)
//   K2'  k_pk_upsweep + k_pk_colscan + k_pk_downsweep: one LSD pass over packed
//                     keys as reduce-then-scan (8-bit digits, ceil(B/8) passes)
//   K3'  k_head_count_pk + k_tile_scan + k_unique_pk: reduce-then-scan of the
//                     head flags on packed keys, unique rows unpacked back to D
//                     words, bucketed (org, new_idx) pairs
//
// Order and equality are preserved exactly: bits dropped by the packing are
// equal in every cleaned row (they equal the replacement key's bits), so the
// first differing bit of two full keys is always a kept bit, kept bits keep
// their relative significance, and unpacking restores the dropped bits from
// the replacement key.
#pragma once

#include "rmx_prep.cuh"

namespace rmx {

template <int KW>
struct PkKey;
template <>
struct PkKey<1> { using T = uint32_t; };
template <>
struct PkKey<2> { using T = uint64_t; };

__device__ __forceinline__ uint32_t low_mask(uint32_t len) { return len >= 32u ? 0xFFFFFFFFu : ((1u << len) - 1u); }

template <int D_CT>
__device__ __forceinline__ uint32_t pick(const uint32_t (&k)[D_CT], uint32_t c) {
    uint32_t w = k[0];
#pragma unroll
    for (int i = 1; i < D_CT; ++i) w = (c == static_cast<uint32_t>(i)) ? k[i] : w;
    return w;
}

__device__ __forceinline__ uint32_t shfl_up_key(uint32_t k) { return __shfl_up_sync(kFull, k, 1); }
__device__ __forceinline__ uint64_t shfl_up_key(uint64_t k) {
    const uint32_t lo = __shfl_up_sync(kFull, static_cast<uint32_t>(k), 1);
    const uint32_t hi = __shfl_up_sync(kFull, static_cast<uint32_t>(k >> 32), 1);
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

// Field-rank tables (rmx_base.cuh) built in shared memory from the K1a field
// sets: rank of every occurring field (pack) or field of every rank (unpack).
__device__ __forceinline__ uint32_t field_rank(const uint32_t* set, uint32_t v) {
    uint32_t r = 0;
    for (uint32_t w = 0; w < (v >> 5); ++w) r += __popc(set[w]);
    return r + __popc(set[v >> 5] & ((1u << (v & 31u)) - 1u));
}

// sentinel: fields outside the set rank as 0xFFFF (k_pack's check of a speculative plan sees the
// overflow above the component's width)
__device__ __forceinline__ void build_field_tables(const uint32_t* fields, const uint32_t* rk, int D, uint16_t* s_rank,
                                                   uint16_t* s_value, bool sentinel = false) {
    for (int c = 0; c < D; ++c) {
        if (!(rk[c] >> 31)) continue;
        const uint32_t* set = fields + c * kFieldWords;
        for (uint32_t v = threadIdx.x; v < static_cast<uint32_t>(kFieldValues); v += blockDim.x) {
            const uint32_t r = field_rank(set, v);
            const bool member = (set[v >> 5] >> (v & 31u)) & 1u;
            if (s_rank) s_rank[c * kFieldValues + v] = static_cast<uint16_t>(sentinel && !member ? 0xFFFFu : r);
            if (s_value && member) s_value[c * kFieldValues + r] = static_cast<uint16_t>(v);
        }
    }
}

// Packed key -> D words: replacement bits outside the varying mask, varying
// bits deposited back from their runs, ranked fields looked up (inverse of k_pack).
template <int D_CT>
__device__ __forceinline__ void unpack_row(uint64_t key, uint32_t* dst, int D, const uint32_t* s_const,
                                           const uint32_t* s_runs, uint32_t nruns, const uint32_t* s_rbeg,
                                           const uint32_t* s_rend, const uint32_t* s_rk, const uint16_t* s_value) {
    if constexpr (D_CT > 0) {
        uint32_t w[D_CT];
#pragma unroll
        for (int c = 0; c < D_CT; ++c) w[c] = s_const[c];
        for (uint32_t q = 0; q < nruns; ++q) {
            const uint32_t* ru = s_runs + 4 * q;
            const uint32_t bits = (static_cast<uint32_t>(key >> ru[3]) & low_mask(ru[2])) << ru[1];
#pragma unroll
            for (int c = 0; c < D_CT; ++c) w[c] |= (ru[0] == static_cast<uint32_t>(c)) ? bits : 0u;
        }
        if constexpr (D_CT <= kMaxRankDim) {
#pragma unroll
            for (int c = 0; c < D_CT; ++c) {
                const uint32_t rk = s_rk[c];
                if (rk >> 31) {
                    const uint32_t r = static_cast<uint32_t>(key >> (rk & 0xFFFFu)) & low_mask((rk >> 16) & 0xFFu);
                    w[c] |= static_cast<uint32_t>(s_value[c * kFieldValues + r]) << kFieldLo;
                }
            }
        }
#pragma unroll
        for (int c = 0; c < D_CT; ++c) dst[c] = w[c];
    } else {
        for (int c = 0; c < D; ++c) {
            uint32_t w = s_const[c];
            for (uint32_t q = s_rbeg[c]; q < s_rend[c]; ++q) {
                const uint32_t* ru = s_runs + 4 * q;
                w |= (static_cast<uint32_t>(key >> ru[3]) & low_mask(ru[2])) << ru[1];
            }
            dst[c] = w;
        }
    }
}

// ---------------------------------------------------------------------------
// K1a: varying bits of the cleaned vertex set.
struct VaryArgs {
    const uint32_t* vtx;
    const uint8_t* flags;
    const uint32_t* idx;
    uint32_t* vary;  // [D]
    uint32_t* fields;  // [D][kFieldWords] set of occurring sign+exponent fields (D <= kMaxRankDim)
    const uint32_t* status;
    uint32_t n;
    int dim;
    int vec;  // vtx and flags 16-byte aligned
    uint32_t shift;  // > 0: only the sample rows (sample_row), for the guessed plan of the value sets
    // after the value-set pass (k_valueset): vstate bit 0 = it checked the rows against the
    // sample's varying bits and field sets, bit 1 = some row fell outside them.  Checked and
    // clean: the sample's outputs are exact and are copied; otherwise the full K1a runs.
    const uint32_t* vstate;
    const uint32_t* sample_vary;
    const uint32_t* sample_fields;
    const uint32_t* gate;  // the fallback after a failed speculative plan: runs only if *gate & kSpecMiss
};

constexpr uint32_t kVstateChecked = 1u, kVstateMiss = 2u, kVstateRedo = 4u;

// The sample that guesses the value-rank layout: one run of kSampleRun rows in
// every kSampleRun << shift (contiguous reads), at a hashed offset inside its
// period -- a fixed offset aliases with periodic data (a grid stored row by
// row showed the same few columns in every run).
constexpr uint32_t kSampleRun = 256;
__host__ __device__ inline uint64_t sample_count(uint64_t n, uint32_t shift) {
    return ((n >> shift) + kSampleRun) & ~static_cast<uint64_t>(kSampleRun - 1);
}
__host__ __device__ inline uint64_t sample_row(uint64_t s, uint32_t shift) {
    const uint64_t b = s / kSampleRun;
    const uint64_t period = static_cast<uint64_t>(kSampleRun) << shift;
    const uint64_t jitter = shift ? (static_cast<uint32_t>(b * 0x9E3779B1ull) >> 8) % (period - kSampleRun + 1) : 0u;
    return b * period + jitter + (s % kSampleRun);
}

// Occurring sign+exponent fields of one component: a per-thread window of 32
// exponents (one register per sign) centred on a sample word -- the thread's
// first row, or the replacement row when that is zero -- catches real
// geometry; anything outside goes to the block's shared set.
struct FieldSet {
    uint32_t win[2];
    uint32_t lo;  // first exponent of the window
    __device__ __forceinline__ void init(uint32_t sample_word) {
        win[0] = win[1] = 0u;
        const uint32_t e = (sample_word >> kFieldLo) & 255u;
        lo = e > 16u ? min(e - 16u, 224u) : 0u;
    }
    __device__ __forceinline__ void add(uint32_t word, uint32_t* s_set) {
        const uint32_t f = word >> kFieldLo;
        const uint32_t x = (f & 255u) - lo;
        if (x < 32u) {
            if (f >> 8) win[1] |= 1u << x;
            else win[0] |= 1u << x;
        } else {
            atomicOr(s_set + (f >> 5), 1u << (f & 31u));
        }
    }
    // OR this thread's windows into the shared set (words may straddle)
    __device__ __forceinline__ void flush(uint32_t* s_set) const {
#pragma unroll
        for (int sg = 0; sg < 2; ++sg) {
            const uint32_t w = win[sg];
            if (!w) continue;
            const uint32_t f0 = (static_cast<uint32_t>(sg) << 8) + lo;  // field of bit 0
            const uint32_t sh = f0 & 31u;
            atomicOr(s_set + (f0 >> 5), w << sh);
            if (sh) atomicOr(s_set + (f0 >> 5) + 1, w >> (32u - sh));
        }
    }
};

template <int D_CT>
__global__ void __launch_bounds__(kBlock) k_vary(VaryArgs a) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (*a.status) return;  // uniform
    if (a.gate && !(*a.gate & 2u)) return;  // (kSpecMiss)
    const int D = D_CT > 0 ? D_CT : a.dim;
    if (a.vstate) {
        const uint32_t st = *a.vstate;
        if (st == kVstateChecked) {  // checked and clean: the sample's outputs are exact
            if (blockIdx.x == 0) {
                if (threadIdx.x < static_cast<unsigned>(D)) a.vary[threadIdx.x] = a.sample_vary[threadIdx.x];
                if (D <= kMaxRankDim)
                    for (uint32_t i = threadIdx.x; i < static_cast<uint32_t>(D) * kFieldWords; i += kBlock)
                        a.fields[i] = a.sample_fields[i];
            }
            return;
        }
    }
    const uint32_t* repl = a.vtx + static_cast<size_t>(a.idx[0]) * D;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const uint64_t start = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    if constexpr (D_CT > 0) {
        constexpr int kSets = D_CT <= kMaxRankDim ? D_CT : 1;
        __shared__ uint32_t s_fields[kSets * kFieldWords];
        uint32_t ref[D_CT], vor[D_CT];
        FieldSet fs[kSets];
#pragma unroll
        for (int c = 0; c < D_CT; ++c) {
            ref[c] = __ldg(repl + c);
            vor[c] = 0u;
            if (c < kSets) {
                const uint32_t w = start < a.n ? __ldg(a.vtx + start * D_CT + c) : 0u;
                fs[c].init((w & 0x7F800000u) ? w : ref[c]);
            }
        }
        for (uint32_t i = threadIdx.x; i < kSets * kFieldWords; i += kBlock) s_fields[i] = 0u;
        __syncthreads();
        auto note = [&](const uint32_t* k) {
            if constexpr (D_CT <= kMaxRankDim) {
#pragma unroll
                for (int c = 0; c < D_CT; ++c) fs[c].add(k[c], s_fields + c * kFieldWords);
            }
        };
        uint64_t done = 0;
        if (a.shift) {  // sample rows only, 4 in flight per thread
            const uint64_t ns = sample_count(a.n, a.shift);
            constexpr int kB = 4;
            for (uint64_t q0 = start; q0 < ns; q0 += kB * stride) {
                uint32_t k[kB][D_CT];
                bool used[kB];
#pragma unroll
                for (int j = 0; j < kB; ++j) {
                    const uint64_t q = q0 + j * stride;
                    const uint64_t i = sample_row(q, a.shift);
                    const bool ok = q < ns && i < a.n;
                    used[j] = ok && a.flags[i] != 0;
#pragma unroll
                    for (int c = 0; c < D_CT; ++c) k[j][c] = ok ? __ldg(a.vtx + i * D_CT + c) : ref[c];
                }
#pragma unroll
                for (int j = 0; j < kB; ++j) {
                    if (used[j]) {
#pragma unroll
                        for (int c = 0; c < D_CT; ++c) vor[c] |= k[j][c] ^ ref[c];
                        note(k[j]);
                    }
                }
            }
            done = a.n;
        }
        if constexpr (D_CT == 3) {
            if (a.vec && !a.shift) {
                const uint64_t ng = a.n >> 2;
                const uint4* v4 = reinterpret_cast<const uint4*>(a.vtx);
                const uint32_t* f4 = reinterpret_cast<const uint32_t*>(a.flags);
                for (uint64_t g = start; g < ng; g += stride) {
                    const uint4 x = __ldcs(v4 + 3 * g), y = __ldcs(v4 + 3 * g + 1), z = __ldcs(v4 + 3 * g + 2);
                    const uint32_t f = __ldcs(f4 + g);
                    const uint32_t k[4][3] = {{x.x, x.y, x.z}, {x.w, y.x, y.y}, {y.z, y.w, z.x}, {z.y, z.z, z.w}};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if ((f >> (8 * j)) & 255u) {
#pragma unroll
                            for (int c = 0; c < 3; ++c) vor[c] |= k[j][c] ^ ref[c];
                            note(k[j]);
                        }
                    }
                }
                done = ng << 2;
            }
        }
        for (uint64_t i = done + start; i < a.n; i += stride) {
            if (a.flags[i]) {
                uint32_t k[D_CT];
#pragma unroll
                for (int c = 0; c < D_CT; ++c) {
                    k[c] = __ldg(a.vtx + i * D_CT + c);
                    vor[c] |= k[c] ^ ref[c];
                }
                note(k);
            }
        }
#pragma unroll
        for (int c = 0; c < D_CT; ++c) {
            const uint32_t v = __reduce_or_sync(kFull, vor[c]);
            if ((threadIdx.x & 31u) == 0u && v) atomicOr(a.vary + c, v);
        }
        if constexpr (D_CT <= kMaxRankDim) {
#pragma unroll
            for (int c = 0; c < D_CT; ++c) fs[c].flush(s_fields + c * kFieldWords);
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < D_CT * kFieldWords; i += kBlock)
                if (s_fields[i]) atomicOr(a.fields + i, s_fields[i]);
        }
    } else {
        __shared__ uint32_t s_vary[RMX_MAX_DIM];
        if (threadIdx.x < RMX_MAX_DIM) s_vary[threadIdx.x] = 0u;
        __syncthreads();
        for (uint64_t i = start; i < a.n; i += stride) {
            if (a.flags[i]) {
                for (int c = 0; c < D; ++c) {
                    const uint32_t x = __ldg(a.vtx + i * D + c) ^ __ldg(repl + c);
                    if (x) atomicOr(s_vary + c, x);
                }
            }
        }
        __syncthreads();
        if (threadIdx.x < static_cast<unsigned>(D) && s_vary[threadIdx.x]) atomicOr(a.vary + threadIdx.x, s_vary[threadIdx.x]);
    }
}

// The speculative plan failed k_pack's check (kSpecMiss): back to the state before the full
// value-set pass, which the re-run then makes (K1a outputs, value sets and check state cleared).
__global__ void k_spec_reset(const uint32_t* spec, uint32_t* vary, uint32_t* fields, uint32_t* vsets,
                             uint32_t* vstate, int D, const uint32_t* status) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (*status || !(*spec & 2u)) return;
    for (int i = threadIdx.x; i < D; i += blockDim.x) vary[i] = 0u;
    if (D <= kMaxRankDim) {
        for (int i = threadIdx.x; i < D * kFieldWords; i += blockDim.x) fields[i] = 0u;
        for (int i = threadIdx.x; i < D * kValueWords; i += blockDim.x) vsets[i] = 0u;
    }
    if (threadIdx.x == 0) *vstate = 0u;
}

// Soup mode: strictly increasing indices (k_mark: every used row referenced once, in row order --
// triangle soups and their shards) and a packed plan with at least one pass.  Used row o then gets
// the origin "used rows before o", which is its index position, so the map fill writes the output
// indices directly (out_idx[position] = new index; unused rows get origins >= I and are skipped):
// no map, no remap.  *soup = I when on, else 0.
// Hash mode: the same when its first hashed pass stages the vertices itself (raw_ok: float3,
// aligned) -- the origins are made there.
__global__ void k_soup_decide(const uint32_t* plan, const uint32_t* order, uint32_t* soup, uint32_t n_idx, int D,
                              int allow, int raw_ok, const uint32_t* status, const uint32_t* gate) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (threadIdx.x != 0 || *status) return;
    if (gate && !(*gate & 2u)) return;  // the re-plan after a failed speculative plan (kSpecMiss)
    const uint32_t* pk = plan + pk_base(4 * D);
    const bool mode_ok = (pk[0] == 1u && pk[3] != 0u) || (pk[0] == 2u && raw_ok);
    *soup = (allow && !(*order & 1u) && mode_ok) ? n_idx : 0u;
}

// Soup mode: used rows before every tile of the pass that makes the origins (rows tile_rows * t ..:
// the packed sort's tiles, or hash mode's first hashed pass's).  The indices are strictly
// increasing, so that is the lower bound of the tile's first row in them.
__global__ void __launch_bounds__(kBlock) k_soup_prefix(const uint32_t* idx, uint32_t n_idx, const uint32_t* soup,
                                                        uint32_t* prefix, uint64_t n_rows, uint32_t tile_pk,
                                                        uint32_t tile_hash, const uint32_t* plan, int D,
                                                        const uint32_t* status, const uint32_t* gate) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (*status || !*soup) return;
    if (gate && !(*gate & 2u)) return;  // (after a failed speculative plan: kSpecMiss)
    const uint32_t tile_rows = plan[pk_base(4 * D)] == 2u ? tile_hash : tile_pk;
    const uint32_t ntiles = static_cast<uint32_t>((n_rows + tile_rows - 1) / tile_rows);
    const uint32_t stride = gridDim.x * kBlock;
    for (uint32_t t = blockIdx.x * kBlock + threadIdx.x; t < ntiles; t += stride) {
        const uint64_t key = static_cast<uint64_t>(t) * tile_rows;
        uint32_t lo = 0, hi = n_idx;
        while (lo < hi) {
            const uint32_t mid = lo + (hi - lo) / 2;
            if (__ldg(idx + mid) < key) lo = mid + 1;
            else hi = mid;
        }
        prefix[t] = lo;
    }
}

// Cleaned row (D_CT <= kMaxRankDim words) -> packed key, one component at a
// time: component c occupies key bits [lo_c, lo_c + w_c) (rmx_base.cuh), its
// value cv_c is its first run (src0, mask0 -> bit 0 of cv; in registers), any
// further runs of c (rare: a shared-memory loop) and its ranked field (looked
// up in the shared field table, placed at frel).  All in 32-bit arithmetic.
template <int D_CT>
struct RowPacker {
    static_assert(D_CT >= 1 && D_CT <= kMaxRankDim, "per-component packing covers D <= kMaxRankDim");
    uint32_t src0[D_CT], msk0[D_CT], frel[D_CT], fmsk[D_CT], lo[D_CT], xr[D_CT];  // xr: extra runs [xr & 0xFFFF, xr >> 16)
    const uint32_t* s_runs;
    const uint16_t* s_rank;  // [D_CT][kFieldValues]

    __device__ __forceinline__ RowPacker(const uint32_t* plan, const uint32_t* runs, uint32_t nruns, const uint16_t* ranks)
        : s_runs(runs), s_rank(ranks) {
        const uint32_t* rk = plan + pk_rank_base(4 * D_CT);
        const uint32_t* vb = plan + pk_value_base(4 * D_CT);
#pragma unroll
        for (int c = 0; c < D_CT; ++c) {
            const uint32_t l = vb[4 + 4 * c];
            lo[c] = min(l, 63u);
            src0[c] = 0u;
            msk0[c] = 0u;
            uint32_t b = nruns, e = 0;
            for (uint32_t r = 0; r < nruns; ++r) {
                if (runs[4 * r] != static_cast<uint32_t>(c)) continue;
                if (b == nruns) {  // the component's first run sits at its low bit
                    b = r;
                    src0[c] = runs[4 * r + 1];
                    msk0[c] = low_mask(runs[4 * r + 2]);
                }
                e = r + 1;
            }
            xr[c] = b < e ? ((b + 1) | (e << 16)) : 0u;
            const bool ranked = rk[c] >> 31;
            frel[c] = ranked ? (rk[c] & 0xFFFFu) - l : 0u;
            fmsk[c] = ranked ? 0xFFFFFFFFu : 0u;  // branch-free: the table entry is masked off
        }
    }

    // no value bits at all (k_valueset: components that are not candidates)
    __device__ __forceinline__ void clear(int c) {
        msk0[c] = 0u;
        fmsk[c] = 0u;
        xr[c] = 0u;
    }

    __device__ __forceinline__ uint32_t value(int c, uint32_t w) const {
        uint32_t v = (w >> src0[c]) & msk0[c];
        for (uint32_t q = xr[c] & 0xFFFFu; q < (xr[c] >> 16); ++q) {
            const uint32_t* ru = s_runs + 4 * q;
            v |= ((w >> ru[1]) & low_mask(ru[2])) << (ru[3] - lo[c]);
        }
        return v | ((static_cast<uint32_t>(s_rank[c * kFieldValues + (w >> kFieldLo)]) << frel[c]) & fmsk[c]);
    }

    __device__ __forceinline__ uint64_t operator()(const uint32_t (&k)[D_CT]) const {
        uint64_t key = 0;
#pragma unroll
        for (int c = 0; c < D_CT; ++c) key |= static_cast<uint64_t>(value(c, k[c])) << lo[c];
        return key;
    }
};

// Inverse of RowPacker: component value cv -> the component's word (the
// replacement row's bits outside the varying mask, the first run and any
// further runs deposited back, the ranked field looked up in the inverse field
// table).
template <int D_CT>
struct RowUnpacker {
    static_assert(D_CT >= 1 && D_CT <= kMaxRankDim, "per-component unpacking covers D <= kMaxRankDim");
    uint32_t src0[D_CT], msk0[D_CT], frel[D_CT], fmask[D_CT], lo[D_CT], xr[D_CT], cst[D_CT];
    bool ranked[D_CT];
    const uint32_t* s_runs;
    const uint16_t* s_value;  // [D_CT][kFieldValues] field of every field rank

    __device__ __forceinline__ RowUnpacker(const uint32_t* plan, const uint32_t* runs, uint32_t nruns,
                                           const uint16_t* values, const uint32_t* s_const)
        : s_runs(runs), s_value(values) {
        const uint32_t* rk = plan + pk_rank_base(4 * D_CT);
        const uint32_t* vb = plan + pk_value_base(4 * D_CT);
#pragma unroll
        for (int c = 0; c < D_CT; ++c) {
            const uint32_t l = vb[4 + 4 * c];
            lo[c] = min(l, 63u);
            src0[c] = 0u;
            msk0[c] = 0u;
            uint32_t b = nruns, e = 0;
            for (uint32_t r = 0; r < nruns; ++r) {
                if (runs[4 * r] != static_cast<uint32_t>(c)) continue;
                if (b == nruns) {
                    b = r;
                    src0[c] = runs[4 * r + 1];
                    msk0[c] = low_mask(runs[4 * r + 2]);
                }
                e = r + 1;
            }
            xr[c] = b < e ? ((b + 1) | (e << 16)) : 0u;
            ranked[c] = rk[c] >> 31;
            frel[c] = ranked[c] ? (rk[c] & 0xFFFFu) - l : 0u;
            fmask[c] = ranked[c] ? low_mask((rk[c] >> 16) & 0xFFu) : 0u;
            cst[c] = s_const[c];
        }
    }

    __device__ __forceinline__ uint32_t word(int c, uint32_t v) const {
        uint32_t w = cst[c] | ((v & msk0[c]) << src0[c]);
        for (uint32_t q = xr[c] & 0xFFFFu; q < (xr[c] >> 16); ++q) {
            const uint32_t* ru = s_runs + 4 * q;
            w |= ((v >> (ru[3] - lo[c])) & low_mask(ru[2])) << ru[1];
        }
        if (ranked[c]) w |= static_cast<uint32_t>(s_value[c * kFieldValues + ((v >> frel[c]) & fmask[c])]) << kFieldLo;
        return w;
    }
};

// ---------------------------------------------------------------------------
// Value ranks (rmx_base.cuh): the layout of each component in the packed key
// before and after, the transform k_pack applies and k_unpack_pk inverts.
template <int D_CT>
struct ValueMap {
    static constexpr int kN = (D_CT > 0 && D_CT <= kMaxRankDim) ? D_CT : 1;
    uint32_t lo[kN], w[kN], nlo[kN], nw[kN];
    uint32_t ranked;  // bit c: component c carries its value rank
    bool on;

    __device__ __forceinline__ void load(const uint32_t* plan) {
        on = false;
        ranked = 0u;
        if constexpr (D_CT > 0 && D_CT <= kMaxRankDim) {
            const uint32_t* vb = plan + pk_value_base(4 * D_CT);
            on = vb[0] == 2u;
#pragma unroll
            for (int c = 0; c < D_CT; ++c) {
                const uint32_t* e = vb + 4 + 4 * c;
                w[c] = e[1];
                nw[c] = e[3] & 0xFFFFu;
                lo[c] = min(e[0], 63u);  // a zero-width component may sit at bit 64
                nlo[c] = min(e[2], 63u);
                ranked |= (e[3] >> 31) << c;
            }
        }
    }
    // key with value ranks from the component values (rank16: [c][2^kMaxValueBits] rank of every occurring value)
    template <int DP>
    __device__ __forceinline__ uint64_t ranked_key(const RowPacker<DP>& pack, const uint32_t (&k)[DP],
                                                   const uint16_t* __restrict__ rank16) const {
        uint64_t out = 0;
#pragma unroll
        for (int c = 0; c < DP; ++c) {
            uint32_t v = pack.value(c, k[c]);
            if ((ranked >> c) & 1u) v = __ldg(rank16 + (static_cast<size_t>(c) << kMaxValueBits) + v);
            out |= static_cast<uint64_t>(v) << nlo[c];
        }
        return out;
    }
    // k_pack under a speculative plan (k_value_plan: sample-saturated value sets, the sample's
    // varying bits and field sets): the key as ranked_key / the plain packing, and in `miss` any
    // sign that the row lies outside what the plan was made from -- a varying bit outside vmask, a
    // field outside the field set (sentinel rank: bits above the component's width), a value
    // outside the value set (rank 0xFFFF)
    template <int DP>
    __device__ __forceinline__ uint64_t checked_key(const RowPacker<DP>& pack, const uint32_t (&k)[DP],
                                                    const uint16_t* __restrict__ rank16, const uint32_t (&ref)[DP],
                                                    const uint32_t (&rmask)[DP], uint32_t (&vor)[DP],
                                                    uint32_t (&vacc)[DP], uint32_t (&rmax)[DP]) const {
        // (value ranks are on: k_value_plan fails a speculative plan that ends without them).  The
        // check only accumulates here -- bits that differ from the replacement row, value bits,
        // the largest rank -- and is decided once per thread (k_pack)
        uint64_t out = 0;
#pragma unroll
        for (int c = 0; c < DP; ++c) {
            uint32_t v = pack.value(c, k[c]);
            vor[c] |= k[c] ^ ref[c];
            vacc[c] |= v;
            // branch-free: components without a value rank read an entry they then ignore
            const uint32_t r = __ldg(rank16 + (static_cast<uint32_t>(c) << kMaxValueBits) + (v & 0xFFFFu));
            rmax[c] = max(rmax[c], r);
            v = (r & rmask[c]) | (v & ~rmask[c]);
            out |= static_cast<uint64_t>(v) << nlo[c];
        }
        return out;
    }
    // inverse (inv: [c][2^kMaxValueBits] value of every rank)
    __device__ __forceinline__ uint64_t from_rank(uint64_t key, const uint16_t* __restrict__ inv) const {
        uint64_t out = 0;
#pragma unroll
        for (int c = 0; c < kN; ++c) {
            uint32_t v = static_cast<uint32_t>(key >> nlo[c]) & low_mask(nw[c]);
            if ((ranked >> c) & 1u) v = __ldg(inv + (static_cast<size_t>(c) << kMaxValueBits) + v);
            out |= static_cast<uint64_t>(v) << lo[c];
        }
        return out;
    }
};

// Shared-memory run list + field-rank table for RowPacker (k_pack, k_valueset).
template <int D_CT>
__device__ __forceinline__ void load_packer(const uint32_t* plan, const uint32_t* fields, uint32_t* s_runs,
                                            uint16_t* s_rank) {
    const int D = D_CT > 0 ? D_CT : 1;
    const uint32_t* pk = plan + pk_base(4 * D);
    for (uint32_t i = threadIdx.x; i < 4 * pk[4]; i += blockDim.x) s_runs[i] = pk[8 + i];
    if constexpr (D_CT > 0 && D_CT <= kMaxRankDim) build_field_tables(fields, plan + pk_rank_base(4 * D_CT), D_CT, s_rank, nullptr);
}

// Occurring packed values of every candidate component over the used rows.
// The packing (the plan argument) is the one guessed from a sample of the rows
// (k_vary over the sample + k_plan): the sample pass (shift > 0) collects the
// sample's values to decide whether value ranks can pay, and the full pass --
// which also computes the exact varying bits and field sets of K1a, so that the
// vertices are read once for both -- collects every used row's values when
// they can.  k_value_plan then keeps a component only if its exact varying bits
// and field set equal the sample's (same packing, so the same values).
// One 1024-thread CTA per SM keeps a byte per possible value (2^w bytes per
// component, <= kValueSetBytes in all: plan_body drops the widest candidates
// beyond that) and sets it with plain stores: lanes that hit the same value
// merge instead of serialising as shared atomics on one bitmap word would
// (structured coordinates crowd a few words).  At the end the bytes are folded
// into bit words and OR-ed into vsets.
struct ValueSetArgs {
    const uint32_t* vtx;
    const uint8_t* flags;
    const uint32_t* idx;     // idx[0]: the replacement row
    const uint32_t* plan;    // the guessed plan (its packing defines the values)
    const uint32_t* fields;  // the field sets it was made from
    uint32_t* vsets;         // [D][kValueWords]
    const uint32_t* guess_vary;  // the sample's varying bits (the full pass checks the rows against them)
    uint32_t* vstate;        // full pass: kVstateChecked | kVstateMiss (for k_vary)
    const uint32_t* status;
    uint32_t n;
    uint32_t shift;          // > 0: the sample rows only (sample_row)
    int vec;
    // second chance (redo != 0): after a miss, collect again with the exact plan (plan = the exact
    // plan, fields = the exact field sets), if the guessed plan (gplan) had found value ranks worth it
    int redo;
    const uint32_t* gplan;
    int parity;              // sample pass: even or odd sample blocks (two sets for the saturation test)
    const uint32_t* spec;    // bit 0: speculative plan (k_value_plan) -- the full pass is not needed
    int fallback;            // the re-run after a failed speculative plan: runs only if kSpecMiss
};

constexpr int kVsThreads = 1024;

template <int D_CT>
__global__ void __launch_bounds__(kVsThreads, 1) k_valueset(ValueSetArgs a) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    static_assert(D_CT >= 1 && D_CT <= kMaxRankDim, "value ranks cover D <= kMaxRankDim");
    uint8_t* s_map = dyn_smem<uint8_t>();  // [sum of 2^w over candidates]
    const uint32_t* pk = a.plan + pk_base(4 * D_CT);
    const uint32_t* vb = a.plan + pk_value_base(4 * D_CT);
    __shared__ uint32_t s_runs[4 * kMaxRuns];
    __shared__ uint16_t s_rank[D_CT * kFieldValues];
    if (*a.status) return;  // uniform
    bool sets;
    if (a.redo) {
        const uint32_t* gvb = a.gplan + pk_value_base(4 * D_CT);
        sets = (*a.vstate & kVstateRedo) && a.gplan[pk_base(4 * D_CT)] != 0u && gvb[0] == 1u && pk[0] != 0u &&
               vb[1] != 0u;
    } else {
        sets = pk[0] == 1u && (a.shift != 0u || vb[0] == 1u) && vb[1] != 0u;
    }
    if (!sets) return;  // (the full pass: k_vary computes K1a's outputs instead)
    if (a.fallback) {
        if (!(*a.spec & 2u)) return;  // (kSpecMiss)
    } else if (!a.redo && a.shift == 0u && a.spec && (*a.spec & 1u)) {
        return;  // speculating: k_pack checks the rows
    }
    // the full pass also checks every used row against the sample's varying bits and field sets
    const bool check = !a.redo && a.vstate != nullptr && a.shift == 0u;
    __shared__ uint32_t s_fset[D_CT * kFieldWords];  // the sample's field sets (check)
    const uint32_t cand = vb[1];
    load_packer<D_CT>(a.plan, a.fields, s_runs, s_rank);
    ValueMap<D_CT> vm;
    vm.load(a.plan);
    uint32_t off[D_CT], vmask[D_CT];
    uint32_t bytes = 0;
#pragma unroll
    for (int c = 0; c < D_CT; ++c) {
        off[c] = bytes;
        vmask[c] = 0u;
        if ((cand >> c) & 1u) {
            bytes += 1u << vm.w[c];
            // a row outside the sample can pack to a wider value (a field above every sampled
            // field ranks to the field count, which needs one more bit when that count is a power
            // of two): such a row sets kVstateMiss and its sets are rebuilt, but its store must
            // stay inside this component's map
            vmask[c] = low_mask(vm.w[c]);
        }
    }
    for (uint32_t i = threadIdx.x; i < bytes / 16u + 1u; i += kVsThreads)
        reinterpret_cast<uint4*>(s_map)[i] = make_uint4(0, 0, 0, 0);
    for (uint32_t i = threadIdx.x; i < D_CT * kFieldWords; i += kVsThreads) s_fset[i] = check ? a.fields[i] : 0u;
    __syncthreads();
    RowPacker<D_CT> pack(a.plan, s_runs, pk[4], s_rank);
    uint32_t gvary[D_CT], miss = 0u;
#pragma unroll
    for (int c = 0; c < D_CT; ++c) gvary[c] = check ? a.guess_vary[c] : 0u;
#pragma unroll
    for (int c = 0; c < D_CT; ++c)
        if (!((cand >> c) & 1u)) {  // value 0 into a spare byte past the maps: no branch per row
            pack.clear(c);
            off[c] = bytes;
        }
    // unused rows stand for the replacement row (used, so its values are in the sets anyway)
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kVsThreads;
    const uint64_t start = static_cast<uint64_t>(blockIdx.x) * kVsThreads + threadIdx.x;
    uint32_t ref[D_CT];
#pragma unroll
    for (int c = 0; c < D_CT; ++c) ref[c] = __ldg(a.vtx + static_cast<size_t>(a.idx[0]) * D_CT + c);
    auto note = [&](const uint32_t (&k)[D_CT], bool used) {
        if (check && used) {
#pragma unroll
            for (int c = 0; c < D_CT; ++c) {
                const uint32_t f = k[c] >> kFieldLo;
                miss |= ((k[c] ^ ref[c]) & ~gvary[c]) | (~(s_fset[c * kFieldWords + (f >> 5)] >> (f & 31u)) & 1u);
            }
        }
#pragma unroll
        for (int c = 0; c < D_CT; ++c) s_map[off[c] + (pack.value(c, used ? k[c] : ref[c]) & vmask[c])] = 1u;
    };
    if (a.shift) {  // the even (parity 0) or odd (parity 1) sample blocks, 4 rows in flight per thread
        const uint64_t ns = sample_count(a.n, a.shift) / 2 + kSampleRun;
        constexpr int kB = 4;
        for (uint64_t q0 = start; q0 < ns; q0 += kB * stride) {
            uint32_t k[kB][D_CT];
            bool ok[kB], used[kB];
#pragma unroll
            for (int j = 0; j < kB; ++j) {
                const uint64_t q = q0 + j * stride;
                const uint64_t qq =
                    (2 * (q / kSampleRun) + static_cast<uint64_t>(a.parity)) * kSampleRun + q % kSampleRun;
                const uint64_t i = sample_row(qq, a.shift);
                ok[j] = q < ns && i < a.n;
                used[j] = ok[j] && a.flags[i] != 0;
#pragma unroll
                for (int c = 0; c < D_CT; ++c) k[j][c] = ok[j] ? __ldg(a.vtx + i * D_CT + c) : ref[c];
            }
#pragma unroll
            for (int j = 0; j < kB; ++j)
                if (ok[j]) note(k[j], used[j]);
        }
    } else {
        uint64_t done = 0;
        if constexpr (D_CT == 3) {
            if (a.vec) {  // 4 rows = 3 x 16 B of vertex words + one flag word per thread iteration
                const uint64_t ng = a.n >> 2;
                const uint4* v4 = reinterpret_cast<const uint4*>(a.vtx);
                const uint32_t* f4 = reinterpret_cast<const uint32_t*>(a.flags);
                auto group = [&](const uint4& x, const uint4& y, const uint4& z, uint32_t f) {
                    const uint32_t k[4][3] = {{x.x, x.y, x.z}, {x.w, y.x, y.y}, {y.z, y.w, z.x}, {z.y, z.z, z.w}};
#pragma unroll
                    for (int j = 0; j < 4; ++j) note(k[j], ((f >> (8 * j)) & 255u) != 0u);
                };
                uint64_t g = start;
                for (; g < ng; g += stride) {
                    if (g + 2 * stride < ng) {  // two iterations ahead
                        prefetch_l2(v4 + 3 * (g + 2 * stride));
                        prefetch_l2(f4 + g + 2 * stride);
                    }
                    group(__ldcs(v4 + 3 * g), __ldcs(v4 + 3 * g + 1), __ldcs(v4 + 3 * g + 2), __ldcs(f4 + g));
                }
                done = ng << 2;
            }
        }
        for (uint64_t i = done + start; i < a.n; i += stride) {
            uint32_t k[D_CT];
#pragma unroll
            for (int c = 0; c < D_CT; ++c) k[c] = __ldg(a.vtx + i * D_CT + c);
            note(k, a.flags[i] != 0);
        }
    }
    if (check) {
        const uint32_t m = __reduce_or_sync(kFull, miss);
        if ((threadIdx.x & 31u) == 0u) atomicOr(a.vstate, kVstateChecked | (m ? kVstateMiss : 0u));
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < D_CT; ++c) {
        if (!((cand >> c) & 1u)) continue;
        const uint32_t words = vm.w[c] > 5u ? (1u << (vm.w[c] - 5u)) : 1u;
        const uint32_t nbytes = 1u << vm.w[c];
        for (uint32_t j = threadIdx.x; j < words; j += kVsThreads) {
            uint32_t x = 0u;
            for (uint32_t q = 0; q < 8u && 4u * (8u * j + q) < nbytes; ++q) {
                const uint32_t b4 = reinterpret_cast<const uint32_t*>(s_map + off[c])[8u * j + q];
#pragma unroll
                for (int e = 0; e < 4; ++e) x |= ((b4 >> (8 * e)) & 1u) << (4u * q + e);
            }
            if (x) atomicOr(a.vsets + c * kValueWords + j, x);
        }
    }
}

// After a miss and the exact K1a: a second chance is needed only if a candidate component's
// packing changed (exact varying bits or field set differ from the sample's) -- misses in other
// components leave the candidates' value sets valid.  If so: kVstateRedo and start the sets over.
__global__ void __launch_bounds__(kBlock) k_vsets_reset(uint32_t* vsets, uint32_t words, uint32_t* vstate,
                                                         const uint32_t* gplan, const uint32_t* vary,
                                                         const uint32_t* svary, const uint32_t* fields,
                                                         const uint32_t* sfields, int D, const uint32_t* status,
                                                         const uint32_t* gate) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    __shared__ uint32_t s_redo;
    if (*status || !(*vstate & kVstateMiss)) return;
    if (gate && !(*gate & 2u)) return;  // the re-run after a failed speculative plan (kSpecMiss)
    if (threadIdx.x == 0) {
        const uint32_t* gvb = gplan + pk_value_base(4 * D);
        bool redo = false;
        if (gplan[pk_base(4 * D)] != 0u && gvb[0] == 1u)
            for (int c = 0; c < D; ++c) {
                if (!((gvb[1] >> c) & 1u)) continue;
                bool same = vary[c] == svary[c];
                for (int w = 0; w < kFieldWords; ++w) same = same && fields[c * kFieldWords + w] == sfields[c * kFieldWords + w];
                redo = redo || !same;
            }
        s_redo = redo ? 1u : 0u;
        if (redo) *vstate |= kVstateRedo;
    }
    __syncthreads();
    if (!s_redo) return;
    for (uint32_t i = threadIdx.x; i < words; i += kBlock) vsets[i] = 0u;
}

// One CTA of 1024 threads.  final == 0 (on the guessed plan, after the sample
// pass): keep the candidates whose sampled value count already needs fewer
// bits, and ask for value sets in the full pass when that alone would shorten
// the key (guessed plan state 1).  final == 1 (on the exact plan, after the full
// pass): keep the candidates packed exactly as guessed, count their values; if
// the key gets shorter, build the rank tables, lay the components out again and
// update the plan (key words, bits, passes, final buffer) -- state 2.
// Otherwise the keys stay as they are.
struct ValuePlanArgs {
    uint32_t* plan;          // decide: the guessed plan; final: the exact plan
    const uint32_t* vsets;
    const uint32_t* vsets_b; // decide after the sample: the odd sample blocks' sets (vsets: the even ones)
    uint16_t* rank16;        // [D][2^kMaxValueBits] rank of every occurring value
    uint16_t* vinv;          // [D][2^kMaxValueBits] value of every rank
    const uint32_t* status;
    int dim;
    int final_pass;
    // final: the guess and what it was made from, against the exact K1a outputs
    const uint32_t* vstate;
    const uint32_t* gplan;
    const uint32_t* svary;
    const uint32_t* sfields;
    const uint32_t* vary;
    const uint32_t* fields;
    // speculation (decide after the sample): when every ranked component's two sample halves saw
    // the same value set and value ranks pay, trust the sample -- no full value-set pass, K1a's
    // outputs copied from the sample (vstate = checked) -- and let k_pack check every row
    // (spec bit 0; a row outside sets bit 1 and the fallback re-plans without value ranks)
    uint32_t* spec;
    uint32_t* spec_vstate;
    int spec_ok;
    int fallback;  // the re-run after a failed speculative plan: runs only if kSpecMiss
};

constexpr uint32_t kSpecOn = 1u, kSpecMiss = 2u;

__device__ __forceinline__ uint32_t bits_for(uint32_t count) { return count <= 1u ? 0u : 32u - __clz(count - 1u); }

__global__ void __launch_bounds__(1024) k_value_plan(ValuePlanArgs a) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    __shared__ uint32_t s_warp[32];
    const int D = a.dim;
    if (*a.status || D > kMaxRankDim) return;
    if (a.fallback && !(*a.spec & kSpecMiss)) return;
    // the second decision (on the full pass's sets) has nothing new when speculating
    if (!a.fallback && !a.final_pass && !a.vsets_b && a.spec && (*a.spec & kSpecOn)) return;
    const bool spec = a.final_pass && a.spec && *a.spec == kSpecOn;  // (not after a miss)
    uint32_t* plan = a.plan;
    uint32_t* pk = plan + pk_base(4 * D);
    uint32_t* vb = plan + pk_value_base(4 * D);
    // a speculative plan must end with value ranks (k_pack's check assumes them): otherwise it
    // counts as failed and the skipped path runs
    auto spec_fail = [&]() {
        if (spec && threadIdx.x == 0) atomicOr(a.spec, kSpecMiss);
    };
    if (pk[0] != 1u) {
        spec_fail();
        return;
    }
    uint32_t cand = vb[1];
    uint32_t unsat = 0u;  // components whose sample halves saw different value sets
    if (a.final_pass) {
        // the value sets hold the guessed packing's values: keep the components packed the same way
        // (after a miss the second chance collected them with the exact packing: all valid)
        const uint32_t* gvb = a.gplan + pk_value_base(4 * D);
        if (a.gplan[pk_base(4 * D)] == 0u || gvb[0] != 1u) {
            spec_fail();
            return;  // uniform
        }
        const bool redone = (*a.vstate & kVstateRedo) != 0u;
        if (!redone) cand &= gvb[1];
        for (int c = 0; c < D && !redone; ++c) {
            bool same = a.vary[c] == a.svary[c];
            for (int w = 0; w < kFieldWords; ++w) same = same && a.fields[c * kFieldWords + w] == a.sfields[c * kFieldWords + w];
            if (!same) cand &= ~(1u << c);
        }
    }
    if (cand == 0u) {
        spec_fail();
        return;  // uniform
    }
    const uint32_t old_bits = pk[2], old_npass = pk[3], old_kw = pk[1];
    uint32_t w[kMaxRankDim], cnt[kMaxRankDim];
    for (int c = 0; c < D; ++c) w[c] = vb[4 + 4 * c + 1];
    __syncthreads();  // every thread has read the plan before thread 0 rewrites it
    const uint32_t t = threadIdx.x;
    for (int c = 0; c < D; ++c) {
        cnt[c] = 0u;
        if (!((cand >> c) & 1u)) continue;
        const uint32_t* set = a.vsets + c * kValueWords;
        uint32_t tot;
        (void)block_exclusive_scan<32>(__popc(set[2 * t]) + __popc(set[2 * t + 1]), s_warp, tot);
        __syncthreads();
        cnt[c] = tot;
        if (a.vsets_b) {
            // two halves of the sample, A (vsets) and B (vsets_b): the number of values that occur is
            // estimated as |A| |B| / |A and B| (capture-recapture) -- a set the sample saturates
            // (lattice axes: both halves see every value) stays small, while ordered data whose
            // halves see different values (grids stored row by row) is not mistaken for one
            const uint32_t* sb = a.vsets_b + c * kValueWords;
            uint32_t nb, ni;
            (void)block_exclusive_scan<32>(__popc(sb[2 * t]) + __popc(sb[2 * t + 1]), s_warp, nb);
            __syncthreads();
            (void)block_exclusive_scan<32>(__popc(sb[2 * t] & set[2 * t]) + __popc(sb[2 * t + 1] & set[2 * t + 1]),
                                           s_warp, ni);
            __syncthreads();
            const uint64_t est = ni ? static_cast<uint64_t>(tot) * nb / ni : (1ull << 32);
            cnt[c] = static_cast<uint32_t>(min(est, static_cast<uint64_t>(0xFFFFFFFFu)));
            if (!(ni == tot && nb == tot)) unsat |= 1u << c;
        }
    }
    uint32_t ranked = 0, nbits = 0;
    for (int c = 0; c < D; ++c) {
        const bool r = ((cand >> c) & 1u) && bits_for(cnt[c]) < w[c];
        if (r) ranked |= 1u << c;
        nbits += r ? bits_for(cnt[c]) : w[c];
    }
    const uint32_t npass = (nbits + 7u) / 8u;
    const bool gain = npass < old_npass || (old_kw == 2u && nbits <= 32u);
    (void)old_bits;
    if (!a.final_pass) {
        if (t == 0) {
            vb[0] = gain ? 1u : 0u;
            vb[1] = gain ? ranked : 0u;
            // speculate only when every varying component has value sets the two sample halves
            // agree on: a component without (too wide, too narrow) gives no sign that the sample
            // saw all of its varying bits and fields (grids stored row by row: the sample's runs
            // see a third of the rows' coordinates)
            uint32_t varying = 0u;
            for (int c = 0; c < D; ++c) varying |= (a.svary && a.svary[c] != 0u ? 1u : 0u) << c;
            if (a.vsets_b && a.spec_ok && gain && (unsat & cand) == 0u && (varying & ~cand) == 0u) {
                // a ranked field at the top of a 32-bit component leaves no room for the sentinel
                const uint32_t* rk = plan + pk_rank_base(4 * D);
                bool room = true;
                for (int c = 0; c < D; ++c)
                    if ((rk[c] >> 31) && vb[4 + 4 * c + 1] >= 32u) room = false;
                if (room) {
                    *a.spec = kSpecOn;
                    *a.spec_vstate = kVstateChecked;
                }
            }
        }
        return;
    }
    if (!gain) {
        if (t == 0) vb[0] = 0u;
        spec_fail();
        return;
    }
    for (int c = 0; c < D; ++c) {
        if (!((ranked >> c) & 1u)) continue;
        const uint32_t* set = a.vsets + c * kValueWords;
        const uint32_t s0 = set[2 * t], s1 = set[2 * t + 1];
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan<32>(__popc(s0) + __popc(s1), s_warp, tot);
        __syncthreads();
        uint16_t* inv = a.vinv + (static_cast<size_t>(c) << kMaxValueBits);
        uint16_t* rnk = a.rank16 + (static_cast<size_t>(c) << kMaxValueBits);
        uint32_t r = ex;
        if (spec) {  // every value below 2^w: its rank, or 0xFFFF outside the set (k_pack's check)
            __shared__ uint32_t s_pre[kValueWords];
            s_pre[2 * t] = ex;
            s_pre[2 * t + 1] = ex + __popc(s0);
            __syncthreads();
            for (uint32_t v = t; v < (1u << w[c]); v += 1024u) {  // coalesced stores
                const uint32_t word = set[v >> 5], bit = 1u << (v & 31u);
                const uint32_t rv = s_pre[v >> 5] + __popc(word & (bit - 1u));
                rnk[v] = (word & bit) ? static_cast<uint16_t>(rv) : static_cast<uint16_t>(0xFFFFu);
                if (word & bit) inv[rv] = static_cast<uint16_t>(v);
            }
            __syncthreads();  // s_pre is reused by the next component
            continue;
        }
        for (uint32_t h = 0; h < 2u; ++h) {
            uint32_t m = h ? s1 : s0;
            while (m) {
                const uint32_t v = ((2u * t + h) << 5) + __ffs(m) - 1u;
                inv[r] = static_cast<uint16_t>(v);
                rnk[v] = static_cast<uint16_t>(r);
                ++r;
                m &= m - 1u;
            }
        }
    }
    if (t == 0) {
        uint32_t run = 0;
        for (int c = D - 1; c >= 0; --c) {
            const bool r = (ranked >> c) & 1u;
            const uint32_t width = r ? bits_for(cnt[c]) : w[c];
            vb[4 + 4 * c + 2] = run;
            vb[4 + 4 * c + 3] = width | (r ? (1u << 31) : 0u);
            run += width;
        }
        pk[1] = run > 32u ? 2u : 1u;
        pk[2] = run;
        pk[3] = npass;
        plan[0] = npass & 1u;
        plan[1] = npass;
        vb[1] = ranked;
        vb[0] = 2u;
    }
}

// ---------------------------------------------------------------------------
// K1b': packed keys + origins, histogram of packed digit 0.
struct PackArgs {
    const uint32_t* vtx;
    const uint8_t* flags;
    const uint32_t* idx;
    const uint32_t* plan;
    uint32_t* buf0;   // keys at word 0, origins at word vals_off
    size_t vals_off;  // words
    uint8_t* digits;  // [n] packed digit 0 per row (read by the first upsweep)
    const uint32_t* fields;  // [D][kFieldWords] occurring sign+exponent fields (K1a)
    const uint16_t* rank16;  // value-rank tables (k_value_plan)
    const uint32_t* status;
    uint32_t n;
    int dim;
    int vec;
    const uint32_t* vary;    // K1a varying bits (the check of a speculative plan)
    uint32_t* spec;          // kSpecOn: check every row against the plan; kSpecMiss: a row failed
    int fallback;            // the re-pack after a failed check (exits unless kSpecMiss)
    uint32_t* win_aux;       // window mode in soup mode: [1] = the replacement row's key (its fallback
                             // gives the unused rows that key back)
};

// CHECK: the variant that packs under a speculative plan and checks every used row (launched
// next to the plain one; each exits unless the plan's state is its own)
template <int D_CT, bool CHECK = false>
__global__ void __launch_bounds__(kBlock, CHECK ? 2 : 4) k_pack(PackArgs a) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    const int D = D_CT > 0 ? D_CT : a.dim;
    const uint32_t* pk = a.plan + pk_base(4 * D);
    __shared__ uint32_t s_runs[4 * kMaxRuns];
    constexpr int kLut = (D_CT > 0 && D_CT <= kMaxRankDim) ? D_CT * kFieldValues : 1;
    __shared__ uint16_t s_rank[kLut];
    if (*a.status || pk[0] != 1u) return;  // uniform (packed mode only)
    if (a.fallback && !(*a.spec & kSpecMiss)) return;  // uniform
    // speculative plan: the CHECK variant packs and checks every used row (D <= kMaxRankDim only:
    // value ranks), the plain one exits
    const bool spec_on = !a.fallback && a.spec && (*a.spec & kSpecOn);
    if (spec_on != CHECK) return;
    constexpr bool check = CHECK && D_CT > 0 && D_CT <= kMaxRankDim;
    const uint32_t nruns = pk[4];
    const bool wide = pk[1] == 2u;
    const uint32_t* rk = a.plan + pk_rank_base(4 * D);
    for (uint32_t i = threadIdx.x; i < 4 * nruns; i += kBlock) s_runs[i] = pk[8 + i];
    if constexpr (D_CT > 0 && D_CT <= kMaxRankDim) build_field_tables(a.fields, rk, D_CT, s_rank, nullptr, check);
    __syncthreads();

    const uint32_t r0 = a.idx[0];
    const uint32_t* repl = a.vtx + static_cast<size_t>(r0) * D;
    uint64_t* keys64 = reinterpret_cast<uint64_t*>(a.buf0);
    uint32_t* keys32 = a.buf0;
    uint32_t* vals = a.buf0 + a.vals_off;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const uint64_t start = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;

    // origins are the row numbers: the first pass makes them itself, so they are
    // only stored when no pass runs (all keys equal)
    const bool want_vals = pk[3] == 0u;
    // the digit of the first executed pass: byte 0, or byte 2 in window mode (rmx_window.cuh)
    const int dshift = pk[6] != 0u ? 16 : 0;
    // window mode in soup mode (pk[6] && !pk[5]): the unused rows stay in the sort but are skipped
    // by origin, so their keys only place them -- a used neighbour's key (the 4-row group) or a
    // hash of the row, never the one replacement key (which would form one giant window)
    const bool spread = pk[6] != 0u && pk[5] == 0u;
    const uint32_t bmask = pk[2] >= 32u ? 0xFFFFFFFFu : (1u << pk[2]) - 1u;
    auto spread_key = [&](uint64_t i) -> uint64_t { return (static_cast<uint32_t>(i) * 0x9E3779B1u) & bmask; };
    auto put = [&](uint64_t i, uint64_t key) {
        if (wide) keys64[i] = key;
        else keys32[i] = static_cast<uint32_t>(key);
        if (want_vals) vals[i] = static_cast<uint32_t>(i);
        a.digits[i] = static_cast<uint8_t>(key >> dshift);
    };

    if constexpr (D_CT > 0) {
        uint32_t ref[D_CT];
#pragma unroll
        for (int c = 0; c < D_CT; ++c) ref[c] = __ldg(repl + c);
        const RowPacker<D_CT> pack0(a.plan, s_runs, nruns, s_rank);
        ValueMap<D_CT> vm;
        vm.load(a.plan);
        // the check's masks: bits outside K1a's varying bits, bits above the component's width (a
        // field outside the field set ranks to the 0xFFFF sentinel), components with value ranks
        uint32_t rmask[D_CT], vor[D_CT], vacc[D_CT], rmax[D_CT];
#pragma unroll
        for (int c = 0; c < D_CT; ++c) {
            rmask[c] = check && ((vm.ranked >> c) & 1u) ? 0xFFFFFFFFu : 0u;
            vor[c] = vacc[c] = rmax[c] = 0u;
        }
        if (check && !vm.on) {  // (k_value_plan marks this case failed already)
            if (threadIdx.x == 0) atomicOr(a.spec, kSpecMiss);
            return;
        }
        auto pack_used = [&](const uint32_t (&k)[D_CT]) -> uint64_t {
            if constexpr (check) return vm.checked_key(pack0, k, a.rank16, ref, rmask, vor, vacc, rmax);
            else return vm.on ? vm.ranked_key(pack0, k, a.rank16) : pack0(k);
        };
        auto pack = [&](const uint32_t (&k)[D_CT]) { return vm.on ? vm.ranked_key(pack0, k, a.rank16) : pack0(k); };
        if (spread && a.win_aux && blockIdx.x == 0 && threadIdx.x == 0) a.win_aux[1] = static_cast<uint32_t>(pack(ref));
        uint64_t done = 0;
        if constexpr (D_CT == 3) {
            if (a.vec) {
                const uint64_t ng = a.n >> 2;
                const uint4* v4 = reinterpret_cast<const uint4*>(a.vtx);
                const uint32_t* f4 = reinterpret_cast<const uint32_t*>(a.flags);
                for (uint64_t g = start; g < ng; g += stride) {
                    if (g + 2 * stride < ng) {  // two iterations ahead
                        prefetch_l2(v4 + 3 * (g + 2 * stride));
                        prefetch_l2(f4 + g + 2 * stride);
                    }
                    const uint4 x = __ldcs(v4 + 3 * g), y = __ldcs(v4 + 3 * g + 1), z = __ldcs(v4 + 3 * g + 2);
                    const uint32_t f = __ldcs(f4 + g);
                    uint32_t k[4][3] = {{x.x, x.y, x.z}, {x.w, y.x, y.y}, {y.z, y.w, z.x}, {z.y, z.z, z.w}};
                    uint64_t key[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const bool used = ((f >> (8 * j)) & 255u) != 0u;
                        if (!used) {
#pragma unroll
                            for (int c = 0; c < 3; ++c) k[j][c] = ref[c];
                        }
                        // (an unused row stands for the replacement row, a used row: checking it is harmless)
                        if constexpr (check) key[j] = pack_used(k[j]);
                        else key[j] = pack(k[j]);
                    }
                    if (spread && f != 0x01010101u) {  // (static indexing only: key[] stays in registers)
                        bool have = false;
                        uint64_t nk = 0u;
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (!have && ((f >> (8 * j)) & 255u) != 0u) {
                                nk = key[j];
                                have = true;
                            }
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (((f >> (8 * j)) & 255u) == 0u) key[j] = have ? nk : spread_key(4 * g + j);
                    }
                    // 16-byte stores of 4 consecutive rows (vals_off is a multiple of 4 words)
                    if (wide) {
                        ulonglong2* k2 = reinterpret_cast<ulonglong2*>(keys64 + 4 * g);
                        __stcs(k2, make_ulonglong2(key[0], key[1]));
                        __stcs(k2 + 1, make_ulonglong2(key[2], key[3]));
                    } else {
                        __stcs(reinterpret_cast<uint4*>(keys32 + 4 * g),
                               make_uint4(static_cast<uint32_t>(key[0]), static_cast<uint32_t>(key[1]),
                                          static_cast<uint32_t>(key[2]), static_cast<uint32_t>(key[3])));
                    }
                    const uint32_t i0 = static_cast<uint32_t>(4 * g);
                    if (want_vals) __stcs(reinterpret_cast<uint4*>(vals + 4 * g), make_uint4(i0, i0 + 1, i0 + 2, i0 + 3));
                    reinterpret_cast<uint32_t*>(a.digits)[g] =
                        (static_cast<uint32_t>(key[0] >> dshift) & 255u) |
                        ((static_cast<uint32_t>(key[1] >> dshift) & 255u) << 8) |
                        ((static_cast<uint32_t>(key[2] >> dshift) & 255u) << 16) |
                        ((static_cast<uint32_t>(key[3] >> dshift) & 255u) << 24);
                }
                done = ng << 2;
            }
        }
        for (uint64_t i = done + start; i < a.n; i += stride) {
            uint32_t k[D_CT];
            const bool used = a.flags[i] != 0;
            if (spread && !used) {
                put(i, spread_key(i));
                continue;
            }
#pragma unroll
            for (int c = 0; c < D_CT; ++c) k[c] = used ? __ldg(a.vtx + i * D_CT + c) : ref[c];
            if constexpr (check) put(i, pack_used(k));
            else put(i, pack(k));
        }
        if constexpr (check) {  // a bit outside K1a's, a field outside the set (sentinel rank: bits
                                // above the width), a value outside the set (rank 0xFFFF)
            uint32_t miss = 0u;
#pragma unroll
            for (int c = 0; c < D_CT; ++c) {
                miss |= vor[c] & ~__ldg(a.vary + c);
                miss |= vm.w[c] < 32u ? vacc[c] >> vm.w[c] : 0u;
                miss |= (rmask[c] && rmax[c] == 0xFFFFu) ? 1u : 0u;
            }
            miss = __reduce_or_sync(kFull, miss);
            if ((threadIdx.x & 31u) == 0u && miss) atomicOr(a.spec, kSpecMiss);
        }
    } else {
        if (spread && a.win_aux && blockIdx.x == 0 && threadIdx.x == 0) {
            uint64_t key = 0;
            for (uint32_t r = 0; r < nruns; ++r) {
                const uint32_t* ru = s_runs + 4 * r;
                key |= static_cast<uint64_t>((__ldg(repl + ru[0]) >> ru[1]) & low_mask(ru[2])) << ru[3];
            }
            a.win_aux[1] = static_cast<uint32_t>(key);
        }
        for (uint64_t i = start; i < a.n; i += stride) {
            if (spread && !a.flags[i]) {
                put(i, spread_key(i));
                continue;
            }
            const uint32_t* row = a.flags[i] ? a.vtx + i * D : repl;
            uint64_t key = 0;
            for (uint32_t r = 0; r < nruns; ++r) {
                const uint32_t* ru = s_runs + 4 * r;
                key |= static_cast<uint64_t>((__ldg(row + ru[0]) >> ru[1]) & low_mask(ru[2])) << ru[3];
            }
            put(i, key);
        }
    }
}

// ---------------------------------------------------------------------------
// Memory-lean mode (rmx_reindex_lean): the plan must be packed (the vertex buffer becomes the
// second sort buffer, 12 bytes per row: at most u64 keys + u32 origins), and the replacement row
// is kept for k_unpack_pk; repl[RMX_MAX_DIM] = 0 stands for its index.
__global__ void k_lean_prepare(const uint32_t* plan, const uint32_t* vtx, const uint32_t* idx, uint32_t* repl,
                               int dim, uint32_t* status) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (*status) return;
    const uint32_t r0 = idx[0];
    for (int c = threadIdx.x; c < dim; c += blockDim.x) repl[c] = vtx[static_cast<size_t>(r0) * dim + c];
    if (threadIdx.x == 0) {
        repl[RMX_MAX_DIM] = 0u;
        if (plan[pk_base(4 * dim)] != 1u) atomicOr(status, RMX_STATUS_LEAN_UNSUPPORTED);
    }
}

// ---------------------------------------------------------------------------
// K2': one LSD pass over (packed key, origin) pairs, as reduce-then-scan:
//   k_pk_upsweep   per-tile digit counts, reading the keys only
//                  (counts stored digit-major: counts[d][tile])
//   k_pk_colscan   one CTA per digit: exclusive scan of counts[d][*] in place,
//                  totals[d]; with the exclusive scan of totals this gives the
//                  global output row of every (digit, tile) run
//   k_pk_downsweep one tile per CTA, no cross-tile dependency: TMA bulk
//                  staging of keys + origins, stable warp multi-split ranking,
//                  slot-index reorder, coalesced write-out
// Measured on B200 the single-kernel onesweep variant spent ~20% of every
// tile in decoupled look-back round trips (L2 latency under full HBM load);
// the extra key-only read of the upsweep (4-8 B/row) is cheaper.
struct SortPkArgs {
    uint32_t* buf0;
    uint32_t* buf1;
    size_t vals_off;       // words
    const uint32_t* plan;
    uint32_t* counts;      // [256][ntiles] per-tile digit counts -> exclusive column scans
    uint32_t* totals;      // [256] digit totals of this pass
    const uint8_t* digits; // [n] this pass's digit per row (written by k_pack / the previous downsweep)
    uint8_t* digits_out;   // [n] the next pass's digit per row, at the row's output position (the other
                           // of two arrays: a downsweep reads this pass's digits while it writes)
    const uint32_t* status;
    uint32_t n;
    uint32_t ntiles;
    uint32_t cstride;      // row stride of counts: ntiles rounded up to kUpGroup
    int dim;
    int pass;
    int rank_force;        // -1 = choose per pass; else kRankMatch / kRankBallot / kRankAtomic
    // soup mode (k_soup_decide): pass 0 gives used row o the origin "used rows before o" (= its
    // index position) and unused rows I + "unused rows before o", from the used flags and the
    // per-tile used counts (k_soup_prefix)
    const uint32_t* soup;
    const uint32_t* soup_prefix;
    const uint8_t* flags;
    // window mode (rmx_window.cuh): passes 0 and 1 do not run (pass 2 is the first, with the
    // row-number / soup origins); win_fb = 1: the four passes of its fallback (origins staged)
    int win_fb;
    uint32_t* win_rows;   // window mode: the used rows the first window pass keeps (its colscan sums them)
    uint32_t tile_rows;   // rows per downsweep tile
};

// window mode: after its first pass (pass 2, which drops the unused rows -- their map entries are
// never read and the replacement row they stand for is a used row) the packed kernels run over
// *win_rows rows; the host sized grids and arrays for the V vertex slots, which bound it
__device__ __forceinline__ void win_rows_patch(const uint32_t* plan, int D, const uint32_t* win_rows, bool after_first,
                                               uint32_t& n, uint32_t& ntiles, uint32_t tile) {
    if (win_rows && after_first && plan[pk_base(4 * D) + 6] != 0u) {
        n = *win_rows;
        ntiles = (n + tile - 1u) / tile;
    }
}
// window mode's first pass when it drops the unused rows (pk[5]: no soup mode)
__device__ __forceinline__ bool win_first_pass(const SortPkArgs& a) {
    return !a.win_fb && a.pass == 2 && a.plan[pk_base(4 * a.dim) + 6] != 0u && a.plan[pk_base(4 * a.dim) + 5] != 0u;
}
__device__ __forceinline__ bool win_after_first(const SortPkArgs& a) {
    return a.win_fb || (a.pass > 2 && a.plan[pk_base(4 * a.dim) + 6] != 0u);
}

// The words a packed pass's kernels test before they start, loaded in one batch (independent
// loads: one L2 round trip in the prologue instead of a chain of them).
struct PkGate {
    uint32_t status, p0, p1, p3, p5, p6, p7, win_rows, soup;
};
__device__ __forceinline__ PkGate pk_gate(const SortPkArgs& a) {
    const uint32_t* pk = a.plan + pk_base(4 * a.dim);
    PkGate g;
    g.status = *a.status;
    g.p0 = pk[0];
    g.p1 = pk[1];
    g.p3 = pk[3];
    g.p5 = pk[5];
    g.p6 = pk[6];
    g.p7 = pk[7];
    g.win_rows = a.win_rows ? *a.win_rows : 0u;
    g.soup = a.soup ? *a.soup : 0u;
    return g;
}
// the pass runs: packed mode, pass < packed passes; window mode runs passes 2 and 3 (its fallback
// passes only when the fallback word is set)
__device__ __forceinline__ bool gate_active(const PkGate& g, const SortPkArgs& a) {
    if (g.status != 0u || g.p0 == 0u || static_cast<uint32_t>(a.pass) >= g.p3) return false;
    if (a.win_fb) return g.p6 != 0u && g.p7 != 0u;
    return !(g.p6 != 0u && a.pass < 2);
}
// window mode's first pass when it drops the unused rows (pk[5]: no soup mode)
__device__ __forceinline__ bool gate_drop(const PkGate& g, const SortPkArgs& a) {
    return !a.win_fb && a.pass == 2 && g.p6 != 0u && g.p5 != 0u;
}
// window mode after its first pass: the kernels run over *win_rows rows
__device__ __forceinline__ void gate_rows(const PkGate& g, SortPkArgs& a, uint32_t tile) {
    if (a.win_rows && g.p6 != 0u && (a.win_fb || a.pass > 2)) {
        a.n = g.win_rows;
        a.ntiles = (a.n + tile - 1u) / tile;
    }
}

// The upsweep counts kUpGroup consecutive tiles per CTA iteration so every digit's
// counts of the group leave as one 32-byte sector (digit-major layout).
constexpr uint32_t kUpGroup = 8;

// true when this packed pass runs (packed mode, pass < number of packed passes)
__device__ __forceinline__ bool pk_pass_active(const SortPkArgs& a) {
    const uint32_t* pk = a.plan + pk_base(4 * a.dim);
    if (pk[0] == 0u || static_cast<uint32_t>(a.pass) >= pk[3]) return false;
    const bool win = pk[6] != 0u;
    if (a.win_fb) return win && pk[7] != 0u;  // window mode's fallback passes
    return !(win && a.pass < 2);              // window mode: passes 2 and 3 only
}

// Per-tile digit counts from the digit-byte array (1 B/row instead of the 4-8 B
// key: k_pack and every downsweep also emit the next pass's digit per row),
// 16 digits per 16-byte load, kUpGroup tiles per CTA iteration.
// DROP: window mode's first pass without soup mode counts the used rows only (its own
// instantiation, as the downsweep's)
template <bool DROP = false>
__global__ void __launch_bounds__(kBlock) k_pk_upsweep(SortPkArgs a0, uint32_t tile_rows) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    SortPkArgs a = a0;
    const PkGate gt = pk_gate(a);
    if (!gate_active(gt, a) || gate_drop(gt, a) != DROP) return;
    gate_rows(gt, a, tile_rows);
    constexpr bool drop = DROP;
    __shared__ uint32_t s_h[kUpGroup * 256];
    const uint32_t ngroups = (a.ntiles + kUpGroup - 1u) / kUpGroup;
    const uint4* d16 = reinterpret_cast<const uint4*>(a.digits);  // tile_rows is a multiple of 16
    for (uint32_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
        for (uint32_t i = threadIdx.x; i < kUpGroup * 256u; i += kBlock) s_h[i] = 0u;
        __syncthreads();
        const uint64_t base = static_cast<uint64_t>(g) * kUpGroup * tile_rows;
        const uint32_t span = static_cast<uint32_t>(min(static_cast<uint64_t>(kUpGroup) * tile_rows,
                                                        static_cast<uint64_t>(a.n) - base));
        const uint32_t span16 = span & ~15u;
#pragma unroll 2
        for (uint32_t r = 16u * threadIdx.x; r < span16; r += 16u * kBlock) {
            const uint4 w = __ldcs(d16 + ((base + r) >> 4));
            uint32_t* h = s_h + (r / tile_rows) * 256u;  // the 16 rows share a tile
            const uint32_t q[4] = {w.x, w.y, w.z, w.w};
            if constexpr (drop) {
                const uint4 f = __ldcs(reinterpret_cast<const uint4*>(a.flags) + ((base + r) >> 4));
                const uint32_t fq[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        if ((fq[k] >> (8 * b)) & 255u) atomicAdd(h + ((q[k] >> (8 * b)) & 255u), 1u);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    atomicAdd(h + (q[k] & 255u), 1u);
                    atomicAdd(h + ((q[k] >> 8) & 255u), 1u);
                    atomicAdd(h + ((q[k] >> 16) & 255u), 1u);
                    atomicAdd(h + (q[k] >> 24), 1u);
                }
            }
        }
        for (uint32_t r = span16 + threadIdx.x; r < span; r += kBlock)
            if (!drop || a.flags[base + r]) atomicAdd(s_h + (r / tile_rows) * 256u + a.digits[base + r], 1u);
        __syncthreads();
        const uint32_t d = threadIdx.x;
        uint4* dst = reinterpret_cast<uint4*>(a.counts + static_cast<size_t>(d) * a.cstride + g * kUpGroup);
        dst[0] = make_uint4(s_h[d], s_h[256 + d], s_h[512 + d], s_h[768 + d]);
        dst[1] = make_uint4(s_h[1024 + d], s_h[1280 + d], s_h[1536 + d], s_h[1792 + d]);
        __syncthreads();
    }
}

// One CTA per digit: exclusive scan of counts[d][0 .. ntiles) in place,
// totals[d].  Chunks of 4096 values: each thread scans 4 consecutive values
// (one coalesced 16-byte access), a block scan joins the threads, a running
// carry joins the chunks.
__global__ void __launch_bounds__(1024) k_pk_colscan(SortPkArgs a0) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    SortPkArgs a = a0;
    const PkGate gt = pk_gate(a);
    if (!gate_active(gt, a)) return;
    gate_rows(gt, a, a.tile_rows);
    __shared__ uint32_t s_warp[32];
    uint32_t* row = a.counts + static_cast<size_t>(blockIdx.x) * a.cstride;
    uint32_t carry = 0;
    for (uint32_t c0 = 0; c0 < a.ntiles; c0 += 4096u) {
        const uint32_t i = c0 + 4u * threadIdx.x;
        uint32_t v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = (i + k < a.ntiles) ? row[i + k] : 0u;
        const uint32_t sum = v[0] + v[1] + v[2] + v[3];
        uint32_t tot;
        uint32_t run = carry + block_exclusive_scan<32>(sum, s_warp, tot);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (i + k < a.ntiles) row[i + k] = run;
            run += v[k];
        }
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.totals[blockIdx.x] = carry;
        if (gate_drop(gt, a) && carry) atomicAdd(a.win_rows, carry);  // the rows the window passes keep
    }
}

template <int IPT>
struct SortPkTraits {
    static constexpr int kTile = kBlock * IPT;
    static __host__ __device__ size_t smem_bytes() {
        // keys sized for u64, origins, slot index, warp counters + peer masks, digit tables, misc, barrier
        // (no peer-mask table: packed passes rank with match or ballots only)
        return static_cast<size_t>(kTile) * (8 + 4 + 2) + (kWarps * 256 + 256 + kWarps + 8) * 4 + 16;
    }
};

// Soup mode, pass 0: the origin of every row of the tile into s_vals (the pass stages keys only):
// used row o -> used rows before o (its index position), unused row o -> I + unused rows before o.
// The tile's used flags were staged into s_flags with the keys.  Thread t takes rows t*IPT ..
// (t+1)*IPT - 1: byte-parallel counts, one block scan, branch-free origins (the downsweep body has
// no predicate registers to spare).
template <int IPT>
__device__ __forceinline__ void soup_origins(const SortPkArgs& a, uint32_t* s_vals, const uint8_t* s_flags,
                                             uint32_t* s_warp, uint32_t base, uint32_t tile_n, uint32_t tile) {
    static_assert(IPT % 4 == 0, "whole flag words per thread");
    constexpr int NW = IPT / 4;
    const uint32_t r0 = threadIdx.x * IPT;
    const uint32_t* f32 = reinterpret_cast<const uint32_t*>(s_flags) + threadIdx.x * NW;
    uint32_t w[NW], cnt = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        // nonzero bytes -> 0x01 per byte; rows at or past tile_n count as unused
        const uint32_t x = f32[i];
        const uint32_t nz = (((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;
        const uint32_t p0 = r0 + 4u * i;
        const uint32_t keep = p0 + 4u <= tile_n ? 0xFFFFFFFFu : (p0 >= tile_n ? 0u : (1u << (8u * (tile_n - p0))) - 1u);
        w[i] = (nz >> 7) & keep;
        cnt += __popc(w[i]);
    }
    uint32_t tot;
    uint32_t before = a.soup_prefix[tile] + block_exclusive_scan<kWarps>(cnt, s_warp, tot);
    const uint32_t un0 = *a.soup + base;  // unused row p: I + (base + p - used rows before p)
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t u = (w[i] >> (8 * j)) & 1u;
            const uint32_t p = r0 + 4u * i + j;
            o[j] = u * before + (1u - u) * (un0 + p - before);
            before += u;
        }
        reinterpret_cast<uint4*>(s_vals + r0)[i] = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

// DROP: window mode's first pass without soup mode keeps the used rows only (a separate
// instantiation: the extra code costs the common passes registers)
template <int KW, int IPT, bool DROP>
__device__ __forceinline__ void sort_pk_body(const SortPkArgs& a, uint32_t* smem, uint32_t tile, uint32_t it, bool iota,
                                             bool soup_on, bool emit_next) {
    using Key = typename PkKey<KW>::T;
    constexpr int TILE = kBlock * IPT;
    const uint32_t src = static_cast<uint32_t>(a.pass) & 1u;
    uint32_t* ib = src ? a.buf1 : a.buf0;
    uint32_t* ob = src ? a.buf0 : a.buf1;
    const Key* __restrict__ in_k = reinterpret_cast<const Key*>(ib);
    const uint32_t* __restrict__ in_v = ib + a.vals_off;
    Key* __restrict__ out_k = reinterpret_cast<Key*>(ob);
    uint32_t* __restrict__ out_v = ob + a.vals_off;
    const int shift = 8 * a.pass;
    // (emit_next: the next pass, if any, reads its digits from the byte array)

    Key* s_keys = reinterpret_cast<Key*>(smem);
    uint32_t* s_vals = smem + static_cast<size_t>(TILE) * 2;  // keys region sized for u64
    uint16_t* s_src = reinterpret_cast<uint16_t*>(s_vals + TILE);
    uint32_t* s_whist = reinterpret_cast<uint32_t*>(s_src + TILE);
    uint32_t* s_gdst = s_whist + kWarps * 256;
    uint32_t* s_warp = s_gdst + 256;
    uint32_t* s_misc = s_warp + kWarps;
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_misc + 8);

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t base = tile * static_cast<uint32_t>(TILE);
    const uint32_t tile_n = min(static_cast<uint32_t>(TILE), a.n - base);
    // pass 0 reads k_pack's keys only: origins are the row numbers (k_pack writes none), or in
    // soup mode the soup origins it makes in s_vals
    // (iota: the first executed pass -- pass 0, or pass 2 in window mode; iota, soup_on and
    // emit_next come from the kernel's prologue, so that no plan load sits between the tile start
    // and its bulk copy)
    constexpr bool drop = DROP;  // window mode's first pass keeps the used rows only
    if (tid == 0) {
        if (it == 0) {
            mbar_init(s_bar, 1);
            fence_mbar_init();
        }
        if (soup_on || drop)  // + the used flags (into the slot-index array, free until the scatter)
            stage_tile2(s_keys, in_k + base, tile_n * static_cast<uint32_t>(sizeof(Key)), s_src, a.flags + base,
                        tile_n, s_bar);
        else if (iota)
            stage_tile(s_keys, in_k + base, tile_n * static_cast<uint32_t>(sizeof(Key)), s_bar);
        else
            stage_tile2(s_keys, in_k + base, tile_n * static_cast<uint32_t>(sizeof(Key)), s_vals, in_v + base,
                        tile_n * 4u, s_bar);
    }
    // global row of this tile's digit-d run = (rows with smaller digits) + (digit-d rows of earlier tiles)
    const uint32_t tot_d = a.totals[tid];
    const int rank_mode = choose_rank(tot_d, a.rank_force == kRankAtomic ? kRankBallot : a.rank_force);
    uint32_t dummy;
    const uint32_t run_base = block_exclusive_scan<kWarps>(tot_d, s_warp, dummy) +
                              a.counts[static_cast<size_t>(tid) * a.cstride + tile];
    for (int i = tid; i < kWarps * 256; i += kBlock) {
        s_whist[i] = 0u;
    }
    __syncthreads();
    mbar_wait(s_bar, it & 1u);
    if (soup_on) soup_origins<IPT>(a, s_vals, reinterpret_cast<const uint8_t*>(s_src), s_warp, base, tile_n, tile);
    uint32_t pk[IPT];
    uint32_t used_mask = 0u;  // drop: bit r = row of round r is used
    if (drop) {  // unused rows take no slot (digit 256)
        const uint8_t* s_fl = reinterpret_cast<const uint8_t*>(s_src);
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
            const bool u = p < tile_n && s_fl[p] != 0;
            used_mask |= (u ? 1u : 0u) << r;
            pk[r] = u ? (static_cast<uint32_t>(s_keys[p] >> shift) & 255u) : 256u;
        }
    }
    if (soup_on || drop) __syncthreads();  // the flags are read before the scatter overwrites s_src
    if (drop) {
        warp_rank<IPT, true>(pk, s_whist + warp * 256, nullptr, rank_mode, true);
    } else if (tile_n == static_cast<uint32_t>(TILE)) {  // full tile: no validity tests
#pragma unroll
        for (int r = 0; r < IPT; ++r)
            pk[r] = static_cast<uint32_t>(s_keys[warp * (32u * IPT) + r * 32u + lane] >> shift) & 255u;
        warp_rank<IPT, false>(pk, s_whist + warp * 256, nullptr, rank_mode, false);
    } else {
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
            pk[r] = p < tile_n ? (static_cast<uint32_t>(s_keys[p] >> shift) & 255u) : 256u;
        }
        warp_rank<IPT, true>(pk, s_whist + warp * 256, nullptr, rank_mode, true);
    }
    __syncthreads();
    {
        const uint32_t d = tid;
        uint32_t wc[kWarps];
        uint32_t cnt = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            wc[w] = s_whist[w * 256 + hsw(d)];
            cnt += wc[w];
        }
        uint32_t tot;
        const uint32_t start = block_exclusive_scan<kWarps>(cnt, s_warp, tot);
        uint32_t run = start;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            s_whist[w * 256 + hsw(d)] = run;  // slot of this warp's first row with digit d
            run += wc[w];
        }
        s_gdst[d] = run_base - start;  // mod 2^32; + tile slot gives the global row
        if (d == 0) s_misc[4] = tot;   // rows ranked in this tile (drop: the used ones)
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
        const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
        if (p < tile_n && (!drop || ((used_mask >> r) & 1u)))
            s_src[s_whist[warp * 256 + (pk[r] >> 16)] + (pk[r] & 0xFFFFu)] = static_cast<uint16_t>(p);
    }
    const uint32_t out_n = drop ? s_misc[4] : tile_n;  // rows this tile writes
    __syncthreads();

    constexpr int U = 4;
    for (uint32_t q0 = tid; q0 < out_n; q0 += U * kBlock) {
        Key k[U];
        uint32_t v[U], dst[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t q = q0 + u * kBlock;
            if (q < out_n) {
                const uint32_t p = s_src[q];
                k[u] = s_keys[p];
                v[u] = iota && !soup_on ? base + p : s_vals[p];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t q = q0 + u * kBlock;
            if (q < out_n) dst[u] = s_gdst[static_cast<uint32_t>(k[u] >> shift) & 255u] + q;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t q = q0 + u * kBlock;
            if (q < out_n) {
                RMX_CHECK_INDEX(dst[u], a.n);
                out_k[dst[u]] = k[u];
                out_v[dst[u]] = v[u];
                if (emit_next) a.digits_out[dst[u]] = static_cast<uint8_t>(k[u] >> (shift + 8));
            }
        }
    }
}

// One tile per CTA, or (tiles_per_cta > 1: the passes that few keys reach, so
// that a pass which does not run costs a small grid) consecutive tiles.
template <int IPT, int MINB, bool DROP = false>
__global__ void __launch_bounds__(kBlock, MINB) k_pk_downsweep(SortPkArgs a0, uint32_t tiles_per_cta) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    SortPkArgs a = a0;
    const PkGate gt = pk_gate(a);
    if (!gate_active(gt, a) || gate_drop(gt, a) != DROP) return;
    gate_rows(gt, a, a.tile_rows);
    uint32_t* smem = dyn_smem<uint32_t>();
    const bool wide = gt.p1 == 2u;
    const bool iota = !a.win_fb && a.pass == (gt.p6 != 0u ? 2 : 0);
    const bool soup_on = iota && gt.soup != 0u;
    const bool emit_next = static_cast<uint32_t>(a.pass) + 1u < gt.p3;
    for (uint32_t j = 0; j < tiles_per_cta; ++j) {
        const uint32_t tile = blockIdx.x * tiles_per_cta + j;
        if (tile >= a.ntiles) break;
        if (j) __syncthreads();  // the next tile's bulk copy overwrites the staging buffers
        if constexpr (DROP) sort_pk_body<1, IPT, true>(a, smem, tile, j, iota, soup_on, emit_next);  // (u32 keys)
        else if (wide) sort_pk_body<2, IPT, false>(a, smem, tile, j, iota, soup_on, emit_next);
        else sort_pk_body<1, IPT, false>(a, smem, tile, j, iota, soup_on, emit_next);
    }
}

// ---------------------------------------------------------------------------
// K2' downsweep, slot-exchange version (k_pk_downsweep2, the default).  The
// tile is staged by TMA bulk copies (u32 keys travel as interleaved (key,
// origin) pairs between passes, so one 8-byte row per bulk byte range; the
// first pass stages k_pack's keys, origins = row numbers; the last pass writes
// keys and origins as separate arrays for K3'; u64 keys keep separate arrays).
// Rows are ranked warp-striped (round r of warp w = row w*32*IPT + 32r + lane)
// with the rank mode fixed at compile time, then each thread moves its rows
// from their staged position to their tile slot IN PLACE (all rows read into
// registers, a barrier, all rows stored at their slots) and the tile leaves in
// slot order: per row one linear and one scattered 8-byte shared access, where
// the staged version read keys and origins by a slot->row index (three
// scattered accesses).  NT threads: 512-thread CTAs put 32 warps on an SM for
// the latency-bound ranking chains at the 64 registers two such CTAs allow.
template <int KW, int IPT, int NT>
struct SortPk2Traits {
    static constexpr int kTile = NT * IPT;
    static constexpr int kNW = NT / 32;
    // staged / exchanged rows (u32 key + origin pairs; u64 keys + origins), per-warp digit
    // counters, digit destinations, scan scratch, barrier
    static __host__ __device__ constexpr size_t smem_bytes() {
        return static_cast<size_t>(kTile) * (KW == 1 ? 8 : 12) + (kNW * 256 + 256 + kNW + 8) * 4 + 16;
    }
};

enum : int { kPkInKeys = 0, kPkInPairs = 1, kPkInSoa = 2 };  // pass input: k_pack keys | pairs | arrays
enum : int { kPkOutPairs = 0, kPkOutSoa = 1 };                // pass output: pairs | arrays

// warp_rank with the multi-split strategy fixed at compile time (no register
// pressure from the strategies not taken)
template <int IPT, bool PARTIAL, int MODE>
__device__ __forceinline__ void warp_rank_ct(uint32_t (&pk)[IPT], uint32_t* wh) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
        const uint32_t d = pk[r];
        uint32_t peers;
        if constexpr (MODE == kRankMatch) {
            peers = __match_any_sync(kFull, d);
        } else {
            peers = kFull;
#pragma unroll
            for (int b = 0; b < 8; ++b) bit_plane_and(peers, d, 1u << b);
            if (PARTIAL) peers &= __ballot_sync(kFull, d < 256u);
        }
        const bool valid = !PARTIAL || d < 256u;
        const uint32_t ds = hsw(d & 255u);
        const uint32_t before = valid ? wh[ds] : 0u;
        __syncwarp();
        if (valid && (peers & lt) == 0u) wh[ds] = before + __popc(peers);
        __syncwarp();
        pk[r] = (ds << 16) | (before + __popc(peers & lt));
    }
}

template <int KW, int IPT, int NT, int IN, int OUT, int MODE>
__device__ __forceinline__ void sort_pk2_body(const SortPkArgs& a, uint32_t* smem, uint32_t tile) {
    using Key = typename PkKey<KW>::T;
    using Tr = SortPk2Traits<KW, IPT, NT>;
    constexpr int TILE = Tr::kTile, NW = Tr::kNW;
    const uint32_t src = static_cast<uint32_t>(a.pass) & 1u;
    uint32_t* ib = src ? a.buf1 : a.buf0;
    uint32_t* ob = src ? a.buf0 : a.buf1;
    const int shift = 8 * a.pass;
    const bool emit_next = static_cast<uint32_t>(a.pass) + 1u < a.plan[pk_base(4 * a.dim) + 3];

    // KW == 1: s_p[TILE] pairs (or s_k32[TILE] keys when staging k_pack's keys)
    // KW == 2: s_k[TILE] keys, s_v[TILE] origins
    uint2* s_p = reinterpret_cast<uint2*>(smem);
    uint32_t* s_k32 = smem;
    Key* s_k = reinterpret_cast<Key*>(smem);
    uint32_t* s_v = smem + static_cast<size_t>(TILE) * 2;
    uint32_t* s_wc = smem + static_cast<size_t>(TILE) * (KW == 1 ? 2 : 3);
    uint32_t* s_gdst = s_wc + NW * 256;
    uint32_t* s_warp = s_gdst + 256;
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_warp + NW + 6);  // 8-byte aligned (TILE even)

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t base = tile * static_cast<uint32_t>(TILE);
    const uint32_t tile_n = min(static_cast<uint32_t>(TILE), a.n - base);
    const bool full = tile_n == static_cast<uint32_t>(TILE);
    if (tid == 0) {
        mbar_init(s_bar, 1);
        fence_mbar_init();
        if constexpr (KW == 1 && IN == kPkInPairs)
            stage_tile(s_p, reinterpret_cast<const uint2*>(ib) + base, tile_n * 8u, s_bar);
        else if constexpr (IN == kPkInKeys)
            stage_tile(s_k, reinterpret_cast<const Key*>(ib) + base, tile_n * static_cast<uint32_t>(sizeof(Key)), s_bar);
        else
            stage_tile2(s_k, reinterpret_cast<const Key*>(ib) + base, tile_n * static_cast<uint32_t>(sizeof(Key)),
                        s_v, ib + a.vals_off + base, tile_n * 4u, s_bar);
    }
    // this pass's digit of every row from the digit array (1 byte per row, written by k_pack / the
    // previous pass at the row's position): coalesced loads in flight during the bulk copy, and no
    // shared-memory read of the staged keys for ranking
    uint32_t dg[IPT];
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
        const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
        dg[r] = (full || p < tile_n) ? static_cast<uint32_t>(__ldcs(a.digits + base + p)) : 0u;
    }
    // global row of this tile's digit-d run = (rows with smaller digits) + (digit-d rows of earlier tiles)
    const uint32_t tot_d = tid < 256u ? a.totals[tid] : 0u;
    uint32_t dummy;
    const uint32_t excl_d = block_exclusive_scan<NW>(tot_d, s_warp, dummy);
    const uint32_t run_base = tid < 256u ? excl_d + a.counts[static_cast<size_t>(tid) * a.cstride + tile] : 0u;
    for (uint32_t i = tid; i < NW * 256u; i += NT) s_wc[i] = 0u;
    __syncthreads();
    mbar_wait(s_bar, 0u);

    auto key_at = [&](uint32_t p) -> Key {
        if constexpr (KW == 1 && IN == kPkInPairs) return s_p[p].x;
        else if constexpr (KW == 1) return s_k32[p];
        else return s_k[p];
    };
    uint32_t pk[IPT];
    if (full) {
#pragma unroll
        for (int r = 0; r < IPT; ++r) pk[r] = dg[r];
        warp_rank_ct<IPT, false, MODE>(pk, s_wc + warp * 256);
    } else {
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
            pk[r] = p < tile_n ? dg[r] : 256u;
        }
        warp_rank_ct<IPT, true, MODE>(pk, s_wc + warp * 256);
    }
    __syncthreads();
    if (tid < 256u) {  // per digit: slot of every warp's first row, global destination of the tile's run
        const uint32_t d = tid;
        uint32_t wc[NW];
        uint32_t cnt = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            wc[w] = s_wc[w * 256 + hsw(d)];
            cnt += wc[w];
        }
        uint32_t x = cnt;  // exclusive prefix over the digits: warp scan + the 8 warp totals
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= static_cast<uint32_t>(o)) x += y;
        }
        if (lane == 31u) s_warp[warp] = x;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        uint32_t before = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) before += (static_cast<uint32_t>(w) < warp) ? s_warp[w] : 0u;
        const uint32_t start = before + x - cnt;
        uint32_t run = start;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            s_wc[w * 256 + hsw(d)] = run;
            run += wc[w];
        }
        s_gdst[d] = run_base - start;  // mod 2^32; + tile slot gives the global row
    }
    __syncthreads();
    // every row from its staged position to its tile slot, in place: all reads, a barrier, all writes
    Key rk[IPT];
    uint32_t rv[IPT];
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
        const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
        if (full || p < tile_n) {
            pk[r] = s_wc[warp * 256 + (pk[r] >> 16)] + (pk[r] & 0xFFFFu);
            if constexpr (KW == 1 && IN == kPkInPairs) {
                const uint2 x = s_p[p];
                rk[r] = x.x;
                rv[r] = x.y;
            } else {
                rk[r] = key_at(p);
                if constexpr (IN == kPkInKeys) rv[r] = base + p;
                else rv[r] = s_v[p];
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
        const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
        if (full || p < tile_n) {
            if constexpr (KW == 1) {
                s_p[pk[r]] = make_uint2(static_cast<uint32_t>(rk[r]), rv[r]);
            } else {
                s_k[pk[r]] = rk[r];
                s_v[pk[r]] = rv[r];
            }
        }
    }
    __syncthreads();
    // slot order out: consecutive slots of one digit are consecutive global rows
#pragma unroll 1
    for (uint32_t q = tid; q < tile_n; q += NT) {
        Key key;
        uint32_t val;
        if constexpr (KW == 1) {
            const uint2 x = s_p[q];
            key = x.x;
            val = x.y;
        } else {
            key = s_k[q];
            val = s_v[q];
        }
        const uint32_t dst = s_gdst[static_cast<uint32_t>(key >> shift) & 255u] + q;
        RMX_CHECK_INDEX(dst, a.n);
        if constexpr (KW == 1 && OUT == kPkOutPairs) {
            reinterpret_cast<uint2*>(ob)[dst] = make_uint2(static_cast<uint32_t>(key), val);
        } else {
            reinterpret_cast<Key*>(ob)[dst] = key;
            ob[a.vals_off + dst] = val;
        }
        if (emit_next) a.digits_out[dst] = static_cast<uint8_t>(key >> (shift + 8));
    }
}

template <int KW, int IPT, int NT, int IN, int OUT>
__device__ __forceinline__ void sort_pk2_mode(const SortPkArgs& a, uint32_t* smem, uint32_t tile) {
    // match when at most 16 digit bins are populated over the whole pass (cheap for low-entropy
    // digits), ballots otherwise -- uniform per pass (the digit totals are global)
    const uint32_t h = threadIdx.x < 256u ? a.totals[threadIdx.x] : 0u;
    const int mode = choose_rank(h, a.rank_force == kRankAtomic ? kRankBallot : a.rank_force);
    if (mode == kRankMatch) sort_pk2_body<KW, IPT, NT, IN, OUT, kRankMatch>(a, smem, tile);
    else sort_pk2_body<KW, IPT, NT, IN, OUT, kRankBallot>(a, smem, tile);
}

template <int IPT, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_pk_downsweep2(SortPkArgs a) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (*a.status || !pk_pass_active(a)) return;
    const uint32_t tile = blockIdx.x;
    if (tile >= a.ntiles) return;
    uint32_t* smem = dyn_smem<uint32_t>();
    const uint32_t* pk = a.plan + pk_base(4 * a.dim);
    const bool first = a.pass == 0, last = static_cast<uint32_t>(a.pass) + 1u == pk[3];
    if (pk[1] == 2u) {  // u64 keys: separate key / origin arrays throughout
        if (first) sort_pk2_mode<2, IPT, NT, kPkInKeys, kPkOutSoa>(a, smem, tile);
        else sort_pk2_mode<2, IPT, NT, kPkInSoa, kPkOutSoa>(a, smem, tile);
    } else if (first) {
        if (last) sort_pk2_mode<1, IPT, NT, kPkInKeys, kPkOutSoa>(a, smem, tile);
        else sort_pk2_mode<1, IPT, NT, kPkInKeys, kPkOutPairs>(a, smem, tile);
    } else {
        if (last) sort_pk2_mode<1, IPT, NT, kPkInPairs, kPkOutSoa>(a, smem, tile);
        else sort_pk2_mode<1, IPT, NT, kPkInPairs, kPkOutPairs>(a, smem, tile);
    }
}

// ---------------------------------------------------------------------------
// K3' as reduce-then-scan (no look-back chain):
//   k_head_count_pk  heads per tile (reads keys only)
//   k_tile_scan      exclusive scan of the per-tile counts, total -> new_count
//   k_unique_pk      one tile per CTA: new index per slot, unique rows unpacked
//                    to D words, bucketed (org, new_idx) pairs (see rmx_unique.cuh)
struct HeadCountArgs {
    uint32_t* buf0;
    uint32_t* buf1;
    const uint32_t* plan;
    uint32_t* counts;  // [ntiles]
    const uint32_t* status;
    uint32_t n;
    uint32_t ntiles;
    uint32_t tile;     // rows per tile
    int dim;
    const uint32_t* win_rows;  // window mode's fallback: the rows its passes kept
};

template <int KW>
__device__ __forceinline__ void head_count_body(const HeadCountArgs& a) {
    using Key = typename PkKey<KW>::T;
    const Key* __restrict__ keys = reinterpret_cast<const Key*>(a.plan[0] ? a.buf1 : a.buf0);
    __shared__ uint32_t s_red[kWarps];
    for (uint32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
        const uint64_t base = static_cast<uint64_t>(t) * a.tile;
        const uint64_t end = min(base + a.tile, static_cast<uint64_t>(a.n));
        uint32_t cnt = 0;
        uint64_t from = base;
        if constexpr (KW == 1) {  // 4 keys per 16-byte load (tiles start at multiples of 4 rows)
            const uint4* k4 = reinterpret_cast<const uint4*>(keys);
            const uint64_t end4 = end & ~static_cast<uint64_t>(3);
#pragma unroll 2
            for (uint64_t g = base + 4u * threadIdx.x; g < end4; g += 4u * kBlock) {
                const uint4 w = __ldg(k4 + (g >> 2));
                cnt += (g == 0 || w.x != __ldg(keys + g - 1)) ? 1u : 0u;
                cnt += (w.y != w.x ? 1u : 0u) + (w.z != w.y ? 1u : 0u) + (w.w != w.z ? 1u : 0u);
            }
            from = max(end4, base);
        }
#pragma unroll 1
        for (uint64_t g = from + threadIdx.x; g < end; g += kBlock)
            cnt += (g == 0 || __ldg(keys + g) != __ldg(keys + g - 1)) ? 1u : 0u;
        cnt = warp_sum(cnt);
        if ((threadIdx.x & 31u) == 0u) s_red[threadIdx.x >> 5] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) tot += s_red[w];
            a.counts[t] = tot;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kBlock) k_head_count_pk(HeadCountArgs a0) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    HeadCountArgs a = a0;
    if (*a.status) return;
    const uint32_t* pk = a.plan + pk_base(4 * a.dim);
    if (pk[0] != 1u || (pk[6] != 0u && pk[7] == 0u)) return;  // packed mode, not window mode
    win_rows_patch(a.plan, a.dim, a.win_rows, true, a.n, a.ntiles, a.tile);
    if (pk[1] == 2u) head_count_body<2>(a);
    else head_count_body<1>(a);
}

// Exclusive scan of per-tile counts in place (one CTA of 1024 threads);
// the total is the output vertex count.
__global__ void __launch_bounds__(1024) k_tile_scan(uint32_t* counts, uint32_t ntiles, const uint32_t* plan, int dim,
                                                    unsigned long long* total_out, const uint32_t* status,
                                                    const uint32_t* win_rows, uint32_t tile) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (*status || plan[pk_base(4 * dim)] != 1u) return;
    if (plan[pk_base(4 * dim) + 6] != 0u && plan[pk_base(4 * dim) + 7] == 0u) return;  // window mode
    uint32_t n_unused = 0;
    win_rows_patch(plan, dim, win_rows, true, n_unused, ntiles, tile);
    __shared__ uint32_t s_warp[32];
    const uint32_t tot = block_scan_counts(counts, ntiles, s_warp);
    if (threadIdx.x == 0) *total_out = tot;
}

struct UniquePkArgs {
    uint32_t* buf0;
    uint32_t* buf1;
    size_t vals_off;
    const uint32_t* plan;
    const uint32_t* prefix; // [ntiles] exclusive head counts
    uint32_t* fill;         // [256]
    const uint32_t* status;
    void* ukeys;            // [U] packed key of every unique row (unpacked by k_unpack_pk)
    uint32_t* sc_org;
    uint8_t* sc_nodup;
    uint32_t* sc_new;
    uint32_t* sc_perm;
    uint32_t n;
    uint32_t ntiles;
    int dim;
    int bucket_shift;
    const uint32_t* win_rows;  // window mode's fallback: the rows its passes kept
    uint32_t n_slots;          // vertex slots V: the extent of the pair buckets (n may be fewer rows)
};

template <int IPT>
struct UniquePkTraits {
    static constexpr int kTile = kBlock * IPT;
    static __host__ __device__ size_t smem_bytes() {
        return static_cast<size_t>(kTile) * (8 + 4 + 8) + (3 * 256 + 2 * kWarps + 8 + 4) * 4 + 16;
    }
};

template <int KW, int IPT>
__device__ __forceinline__ void unique_pk_body(const UniquePkArgs& a, uint32_t* smem) {
    using Key = typename PkKey<KW>::T;
    constexpr int TILE = kBlock * IPT;
    const uint32_t fin = a.plan[0];
    const uint32_t* fb = fin ? a.buf1 : a.buf0;
    const Key* __restrict__ keys = reinterpret_cast<const Key*>(fb);
    const uint32_t* __restrict__ vals = fb + a.vals_off;
    uint2* __restrict__ pairs = reinterpret_cast<uint2*>(fin ? a.buf0 : a.buf1);

    Key* s_keys = reinterpret_cast<Key*>(smem);
    uint32_t* s_vals = smem + static_cast<size_t>(TILE) * 2;
    uint2* s_pairs = reinterpret_cast<uint2*>(s_vals + TILE);
    uint32_t* s_bcnt = reinterpret_cast<uint32_t*>(s_pairs + TILE);
    uint32_t* s_bcur = s_bcnt + 256;
    uint32_t* s_bglob = s_bcur + 256;
    uint32_t* s_warp = s_bglob + 256;
    uint32_t* s_misc = s_warp + 2 * kWarps;
    Key* s_prev = reinterpret_cast<Key*>(s_misc + 8);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_misc + 10);

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const int bs = a.bucket_shift;
    if (tid == 0) {
        mbar_init(s_bar, 1);
        fence_mbar_init();
    }
    Key* __restrict__ ukeys = static_cast<Key*>(a.ukeys);
    // static tile striding: no cross-tile dependency remains (prefixes come from k_tile_scan).
    // The staging buffers are free once phase 1 has moved a tile into registers, so the
    // next tile's bulk copy is issued there and overlaps phase 2 and the pair write-out.
    auto issue = [&](uint32_t t) {
        const uint32_t b = t * static_cast<uint32_t>(TILE);
        const uint32_t n = min(static_cast<uint32_t>(TILE), a.n - b);
        stage_tile2(s_keys, keys + b, n * static_cast<uint32_t>(sizeof(Key)), s_vals, vals + b, n * 4u, s_bar);
        if (t > 0) *s_prev = keys[b - 1];
    };
    if (tid == 0 && blockIdx.x < a.ntiles) issue(blockIdx.x);
    uint32_t it = 0;
    for (uint32_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++it) {
    const uint32_t base = tile * static_cast<uint32_t>(TILE);
    const uint32_t tile_n = min(static_cast<uint32_t>(TILE), a.n - base);
    const uint32_t tile_prefix = a.prefix[tile];  // consumed in phase 2: the load overlaps phase 1
    s_bcnt[tid] = 0u;
    __syncthreads();
    mbar_wait(s_bar, it & 1u);

    // ---- phase 1: head flags (warp-striped rows; the previous key comes from the
    // neighbouring lane), per-warp totals, bucket counts.  Keys and origins stay
    // in registers for phase 2.
    uint32_t bal[IPT];
    Key kreg[IPT];
    uint32_t vreg[IPT];
    uint32_t wtotal = 0;
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
        const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
        const bool valid = p < tile_n;
        const Key key = valid ? s_keys[p] : Key(0);
        Key prev = shfl_up_key(key);
        if (lane == 0 && valid && p > 0) prev = s_keys[p - 1];
        if (lane == 0 && p == 0 && base > 0) prev = *s_prev;
        bool head = false;
        uint32_t org = 0;
        if (valid) {
            head = (base + p == 0u) || key != prev;
            org = s_vals[p];
            atomicAdd(s_bcnt + (org >> bs), 1u);
        }
        kreg[r] = key;
        vreg[r] = org;
        bal[r] = __ballot_sync(kFull, head);
        wtotal += __popc(bal[r]);
    }
    if (lane == 0) s_warp[warp] = wtotal;
    __syncthreads();
    if (tid == 0 && tile + gridDim.x < a.ntiles) issue(tile + gridDim.x);
    uint32_t wexcl = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) wexcl += (static_cast<uint32_t>(w) < warp) ? s_warp[w] : 0u;
    // bucket space of this tile's pairs: the reservation's round trip overlaps phase 2
    const uint32_t bcnt = s_bcnt[tid];
    uint32_t bstart, bfill = 0u;
    {
        uint32_t tot;
        bstart = block_exclusive_scan<kWarps>(bcnt, s_warp + kWarps, tot);
        s_bcur[tid] = bstart;
        if (bcnt) bfill = atomicAdd(a.fill + tid, bcnt);
    }
    __syncthreads();

    // ---- phase 2: new index per slot, bucketed pairs, unique rows out
    uint32_t running = tile_prefix + wexcl;
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
        const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
        if (p < tile_n) {
            const uint32_t nidx = running + __popc(bal[r] & lanemask_le()) - 1u;
            const uint32_t org = vreg[r];
            s_pairs[atomicAdd(s_bcur + (org >> bs), 1u)] = make_uint2(org, nidx);
            const bool head = (bal[r] >> lane) & 1u;
            RMX_CHECK_INDEX(nidx, a.n);
            if (head) ukeys[nidx] = kreg[r];
            if (a.sc_org) a.sc_org[base + p] = org;
            if (a.sc_nodup) a.sc_nodup[base + p] = head ? 1 : 0;
            if (a.sc_new) a.sc_new[base + p] = nidx;
            if (a.sc_perm) a.sc_perm[org] = base + p;
        }
        running += __popc(bal[r]);
    }
    if (bcnt) s_bglob[tid] = (tid << bs) + bfill - bstart;
    __syncthreads();
    // ---- bucket runs out: consecutive slots of one bucket are consecutive pairs
    for (uint32_t q = tid; q < tile_n; q += kBlock) {
        const uint2 pr = s_pairs[q];
        RMX_CHECK_INDEX(s_bglob[pr.x >> bs] + q, a.n_slots);
        pairs[s_bglob[pr.x >> bs] + q] = pr;
    }
    __syncthreads();
    }
}

template <int IPT>
__global__ void __launch_bounds__(kBlock, 3) k_unique_pk(UniquePkArgs a0) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    UniquePkArgs a = a0;
    if (*a.status) return;
    const uint32_t* pk = a.plan + pk_base(4 * a.dim);
    if (pk[0] != 1u || (pk[6] != 0u && pk[7] == 0u)) return;  // packed mode, not window mode
    win_rows_patch(a.plan, a.dim, a.win_rows, true, a.n, a.ntiles, static_cast<uint32_t>(UniquePkTraits<IPT>::kTile));
    uint32_t* smem = dyn_smem<uint32_t>();
    if (pk[1] == 2u) unique_pk_body<2, IPT>(a, smem);
    else unique_pk_body<1, IPT>(a, smem);
}

// Unique rows out: packed key -> D words (dense, one row per thread; the
// unique kernel only stores the packed key of each head).
struct UnpackPkArgs {
    const uint32_t* plan;
    const uint32_t* vtx;    // replacement key source (vtx[idx[0]])
    const uint32_t* idx;
    const uint32_t* vary;
    const uint32_t* fields;
    const void* ukeys;
    const uint16_t* vinv;   // value-rank inverse tables (k_value_plan)
    uint32_t* out_vtx;
    const unsigned long long* count;
    const uint32_t* status;
    int dim;
    int vec;  // out_vtx 16-byte aligned
    // lean mode (rmx_reindex_lean): the output rows go to the final sort buffer (buf0 or buf1 by the
    // plan's parity), and *where records which
    uint32_t* lean_buf0;
    uint32_t* lean_buf1;
    uint32_t* where;
};

template <int D_CT>
__global__ void __launch_bounds__(kBlock, 4) k_unpack_pk(UnpackPkArgs a) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (*a.status) return;
    const int D = D_CT > 0 ? D_CT : a.dim;
    const uint32_t* pk = a.plan + pk_base(4 * D);
    if (pk[0] != 1u) return;  // packed mode only
    __shared__ uint32_t s_runs[4 * kMaxRuns];
    __shared__ uint32_t s_const[RMX_MAX_DIM];  // replacement bits outside the varying mask
    __shared__ uint32_t s_rbeg[RMX_MAX_DIM];   // run range of each component
    __shared__ uint32_t s_rend[RMX_MAX_DIM];
    __shared__ uint32_t s_rk[RMX_MAX_DIM];
    constexpr int kLut = (D_CT > 0 && D_CT <= kMaxRankDim) ? D_CT * kFieldValues : 1;
    __shared__ uint16_t s_value[kLut];
    const uint32_t nruns = pk[4];
    const uint32_t* rk = a.plan + pk_rank_base(4 * D);
    for (uint32_t i = threadIdx.x; i < 4 * nruns; i += kBlock) s_runs[i] = pk[8 + i];
    if constexpr (D_CT > 0 && D_CT <= kMaxRankDim) build_field_tables(a.fields, rk, D_CT, nullptr, s_value);
    if (threadIdx.x < static_cast<uint32_t>(D)) {
        const uint32_t c = threadIdx.x;
        s_rk[c] = rk[c];
        // a ranked field comes back from the value table, not from the replacement row
        const uint32_t keep = (rk[c] >> 31) ? ~(a.vary[c] | ~((1u << kFieldLo) - 1u)) : ~a.vary[c];
        s_const[c] = a.vtx[static_cast<size_t>(a.idx[0]) * D + c] & keep;
        uint32_t b = nruns, e = 0;
        for (uint32_t r = 0; r < nruns; ++r)
            if (pk[8 + 4 * r] == c) {
                b = min(b, r);
                e = r + 1;
            }
        s_rbeg[c] = b < e ? b : 0u;
        s_rend[c] = e;
    }
    __syncthreads();
    const uint64_t U = *a.count;
    const bool wide = pk[1] == 2u;
    if (a.lean_buf0) {
        const uint32_t fin = a.plan[0];
        a.out_vtx = fin ? a.lean_buf1 : a.lean_buf0;
        if (blockIdx.x == 0 && threadIdx.x == 0) *a.where = fin;
    }
    const uint64_t* k64 = static_cast<const uint64_t*>(a.ukeys);
    const uint32_t* k32 = static_cast<const uint32_t*>(a.ukeys);
    ValueMap<D_CT> vm;
    vm.load(a.plan);
    auto load_key = [&](uint64_t i) {
        const uint64_t key = wide ? __ldcs(k64 + i) : static_cast<uint64_t>(__ldcs(k32 + i));
        return vm.on ? vm.from_rank(key, a.vinv) : key;
    };
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    uint64_t done = 0;
    if constexpr (D_CT == 3 || D_CT == 4) {
        if (a.vec) {  // 4 rows per thread, written as D_CT 16-byte stores
            const RowUnpacker<D_CT> up(a.plan, s_runs, nruns, s_value, s_const);
            // key (value ranks inverted per component) -> component value -> word
            auto unpack4 = [&](uint64_t key, uint32_t* w) {
#pragma unroll
                for (int c = 0; c < D_CT; ++c) {
                    uint32_t v;
                    if (vm.on) {
                        v = static_cast<uint32_t>(key >> vm.nlo[c]) & low_mask(vm.nw[c]);
                        if ((vm.ranked >> c) & 1u) v = __ldg(a.vinv + (static_cast<size_t>(c) << kMaxValueBits) + v);
                    } else {
                        v = static_cast<uint32_t>(key >> up.lo[c]) & low_mask(vm.w[c]);
                    }
                    w[c] = up.word(c, v);
                }
            };
            uint32_t w[4 * D_CT];
            const uint64_t ng = U >> 2;
            for (uint64_t g = t0; g < ng; g += stride) {
                uint64_t key[4];  // the group's four keys in one or two 16-byte loads
                if (wide) {
                    const ulonglong2 p0 = __ldcs(reinterpret_cast<const ulonglong2*>(k64) + 2 * g);
                    const ulonglong2 p1 = __ldcs(reinterpret_cast<const ulonglong2*>(k64) + 2 * g + 1);
                    key[0] = p0.x;
                    key[1] = p0.y;
                    key[2] = p1.x;
                    key[3] = p1.y;
                } else {
                    const uint4 p = __ldcs(reinterpret_cast<const uint4*>(k32) + g);
                    key[0] = p.x;
                    key[1] = p.y;
                    key[2] = p.z;
                    key[3] = p.w;
                }
#pragma unroll
                for (int r = 0; r < 4; ++r) unpack4(key[r], w + r * D_CT);
                uint4* dst = reinterpret_cast<uint4*>(a.out_vtx + 4 * g * D_CT);
#pragma unroll
                for (int q = 0; q < D_CT; ++q)
                    __stcs(dst + q, make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]));
            }
            done = ng << 2;
        }
    }
    for (uint64_t i = done + t0; i < U; i += stride) {
        const uint64_t key = load_key(i);
        unpack_row<D_CT>(key, a.out_vtx + i * D, D, s_const, s_runs, nruns, s_rbeg, s_rend, s_rk, s_value);
    }
}

}  // namespace rmx
