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

// ---------------------------------------------------------------------------
// Welded (indexed) tiles of the C4 merge workload (bit-identical to
// oracle/lattice.py:welded_tile): n x n quads whose lattice rows start at
// row0, each point stored once with 5 % unused rows interleaved; points and
// triangles row-major, or (shuffle) at seeded positions / in seeded order.
struct Perm {
    uint64_t n;
    uint32_t half;
    uint64_t mask;
    uint64_t keys[4];
};

inline Perm make_perm(uint64_t n, uint64_t seed) {
    Perm f{};
    f.n = n;
    int bits = 0;
    while ((1ull << bits) < n) ++bits;  // bit length of n-1
    if (bits < 2) bits = 2;
    bits += bits & 1;
    f.half = static_cast<uint32_t>(bits / 2);
    f.mask = (1ull << f.half) - 1;
    for (int r = 0; r < 4; ++r) f.keys[r] = splitmix64(static_cast<uint64_t>(r) + seed * 4 + 1);
    return f;
}

__device__ __forceinline__ uint64_t perm_apply(uint64_t v, const Perm& f) {
    do {
        uint64_t left = v >> f.half, right = v & f.mask;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint64_t g = (splitmix64(right ^ f.keys[r]) >> 7) & f.mask;
            const uint64_t nl = right;
            right = left ^ g;
            left = nl;
        }
        v = (left << f.half) | right;
    } while (v >= f.n);  // cycle walking
    return v;
}

struct TileArgs {
    uint32_t n;        // quads per side
    uint32_t row0;     // global lattice row of local row 0
    int shuffle;       // 0: row-major points and triangles; 1: seeded positions and order
    uint64_t n_pts, n_unused, n_elem;
    Perm pts, elems;
    uint64_t useed;
    uint32_t* vtx;
    uint32_t* idx;
};

__device__ __forceinline__ uint64_t tile_slot(uint64_t q, const TileArgs& a) {
    return q + (q * a.n_unused) / a.n_pts;
}

__global__ void __launch_bounds__(kBlock) k_gen_welded_tile(TileArgs a) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    const uint32_t cols = a.n + 1;
    // points at their positions, unused rows after each position
    for (uint64_t p = t0; p < a.n_pts; p += stride) {
        const uint64_t q = a.shuffle ? perm_apply(p, a.pts) : p;
        const int i = static_cast<int>(a.row0 + p / cols), j = static_cast<int>(p % cols);
        uint32_t* row = a.vtx + tile_slot(q, a) * 3;
        row[0] = __float_as_uint(__fmul_rn(static_cast<float>(i), 0.5f));
        row[1] = __float_as_uint(__fmul_rn(static_cast<float>(j), 0.5f));
        row[2] = __float_as_uint(__fmul_rn(static_cast<float>((7 * i + 13 * j) % 64), 0.25f));
    }
    for (uint64_t q = t0; q < a.n_pts; q += stride) {
        const uint64_t u0 = (q * a.n_unused) / a.n_pts, u1 = ((q + 1) * a.n_unused) / a.n_pts;
        for (uint64_t o = u0; o < u1; ++o) {
            uint32_t* row = a.vtx + (q + u0 + 1 + (o - u0)) * 3;
            for (int c = 0; c < 3; ++c) {
                const uint64_t h = splitmix64((o * 3 + c) ^ a.useed);
                const uint64_t expo = (0x7Full + ((h >> 32) % 10ull)) << 23;
                row[c] = static_cast<uint32_t>((h & 0x807FFFFFull) | expo);
            }
        }
    }
    // triangles: corner points -> their slots
    for (uint64_t e = t0; e < a.n_elem; e += stride) {
        const uint64_t t = a.shuffle ? perm_apply(e, a.elems) : e;
        const uint64_t qd = t >> 1;
        const int h = static_cast<int>(t & 1);
        const uint32_t qi = static_cast<uint32_t>(qd / a.n), qj = static_cast<uint32_t>(qd % a.n);
        const uint32_t ci[3] = {qi, qi + 1, h ? qi : qi + 1};
        const uint32_t cj[3] = {qj, h ? qj + 1 : qj, qj + 1};
        for (int s = 0; s < 3; ++s) {
            const uint64_t p = static_cast<uint64_t>(ci[s]) * cols + cj[s];
            a.idx[e * 3 + s] = static_cast<uint32_t>(tile_slot(a.shuffle ? perm_apply(p, a.pts) : p, a));
        }
    }
}

}  // namespace rmx
