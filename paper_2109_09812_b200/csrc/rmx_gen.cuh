// rmx_gen.cuh -- synthetic lattice soups for the bench (bit-identical to oracle/lattice.py).
#pragma once

#include "rmx_base.cuh"

namespace rmx {

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
    uint64_t e0;      // first element written (element range [e0, take))
    uint64_t v0;      // its first vertex slot; written slots and indices are relative to it
    uint64_t take;    // end of the element range
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
    for (uint64_t e = g.e0 + static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x; e < g.take; e += stride) {
        uint64_t t = feistel(e, g);
        while (t >= g.n_elem) t = feistel(t, g);
        const uint64_t u0 = (e * g.n_unused) / g.n_elem;
        const uint64_t u1 = ((e + 1) * g.n_unused) / g.n_elem;
        const uint64_t base = e * K + u0 - g.v0;
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
            g.idx[(e - g.e0) * K + s] = static_cast<uint32_t>(base + s);
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

// ---------------------------------------------------------------------------
// grid_quads(n) of the paper's Table 1 (reference bench.py:42-68): quad q has
// qi = q mod n, qj = q div n and owns 5 float2 rows -- corners (qi,qj),
// (qi+1,qj), (qi+1,qj+1), (qi,qj+1) and the unused centre (qi+.5,qj+.5) --
// and the element (5q, 5q+1, 5q+2, 5q+3) (uint32 arithmetic, like the
// reference's uint32 arange).  One thread per output word: both arrays are
// written fully coalesced.
__global__ void __launch_bounds__(kBlock) k_gen_grid_quads(uint32_t n, uint64_t quads, uint32_t* vtx,
                                                           uint32_t* idx) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    for (uint64_t w = t0; w < quads * 10u; w += stride) {
        const uint64_t q = w / 10u;
        const uint32_t r = static_cast<uint32_t>(w - q * 10u);
        const float qi = static_cast<float>(q % n), qj = static_cast<float>(q / n);
        const uint32_t row = r >> 1, c = r & 1u;
        const float base = c ? qj : qi;
        float v;
        if (row == 4u) {
            v = __fadd_rn(base, 0.5f);
        } else {
            // corners: x + 1 for rows 1, 2; y + 1 for rows 2, 3
            const bool plus = c ? (row >= 2u) : (row == 1u || row == 2u);
            v = plus ? __fadd_rn(base, 1.0f) : base;
        }
        vtx[w] = __float_as_uint(v);
    }
    for (uint64_t w = t0; w < quads * 4u; w += stride) {
        const uint64_t q = w >> 2;
        idx[w] = static_cast<uint32_t>(q) * 5u + static_cast<uint32_t>(w & 3u);
    }
}

}  // namespace rmx
