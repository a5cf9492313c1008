// rmx_hash.cuh -- wide keys: group by a key hash first, then sort only the
// distinct rows exactly (plan mode 2, "hash").
//
// When more than 64 key bits vary over the cleaned vertex set (real-valued
// geometry: full float mantissas), an LSD sort of the whole vertex set moves
// 16-20-byte rows through 4D byte passes (C2s: 12 passes over 157.5M rows).
// Soups repeat each vertex ~6 times, so most of that work sorts duplicates.
// Hash mode instead
//
//   k_hash_build    cleaned AoS rows (key words, origin) and the histograms of
//                   the top kHashPasses bytes of h = hash_key(row) (rmx_hashfn.cuh)
//   hashed passes   k_sort_pass<..., HASHED>: the rows grouped by the top 24
//                   bits of h -- equal keys land next to each other, in buckets
//                   of ~9 rows (C2s; 16 bits left ~2400-row buckets, which the
//                   2048-row dedup tiles split: 1.8 candidates per key)
//   k_hash_dedup    per tile of kHashTile rows, a shared-memory hash table of
//                   the tile's distinct keys: one *candidate* row (key words,
//                   group id) per distinct key of the tile, (group id, origin)
//                   for every row
//   AoS passes      exact LSD sort of the n_cand candidate rows (k_sort_pass,
//                   bitwise order, constant digits skipped)
//   k_unique        adjacent-compare heads over the sorted candidates: the
//                   output rows, the count, (group, new index) pairs
//   k_map_fill      rank_of[group] = new index
//   k_hash_pairs    (origin, rank_of[group of the row]) pairs bucketed by origin
//   k_map_fill      map[origin] = new index
//
// Every access to the vertex set is a stream or a bucketed multi-split: on B200
// a random gather of a vertex row costs ~128 B of DRAM traffic (4.5 ms for the
// 157.5M rows of C2s, tools/micro/gather_bench.cu), more than the two passes.
//
// Exactness does not depend on the hash: the dedup compares whole keys, a key
// split over two tiles (or hash buckets of a collision) just yields two
// candidates, and the exact sort of the candidates gives both one new index.
// Candidate numbering follows the order in which tiles reserve their range
// (atomic), which never shows in the results.  The scratch arrays of the
// stable sort (org_id, perm) are not produced here: a call that asks for
// scratch takes the AoS path.
#pragma once

#include "rmx_prep.cuh"
#include "rmx_hashfn.cuh"

namespace rmx {

__device__ __forceinline__ bool hash_mode(const uint32_t* plan, int dim) { return plan[pk_base(4 * dim)] == 2u; }

struct HashArgs {
    const uint32_t* vtx;
    const uint8_t* flags;
    const uint32_t* idx;      // idx[0]: the replacement row (pipeline.py:148)
    const uint32_t* plan;
    uint32_t* rows0;          // cleaned rows (the hashed passes ping-pong rows0 / rows1); the grouped
    uint32_t* rows1;          // rows end in buffer kHashPasses & 1, the candidate rows go to the other
    uint32_t* hhist;          // [kHashPasses][256] the hashed digits' histograms
    uint2* grp_org;           // [n] (group id, origin) of every row, in hash-bucket order
    uint32_t* n_cand;         // number of candidate rows (tiles reserve ranges)
    uint32_t* hist;           // [4D][256]: passes 0..3 over the candidate rows
    const uint32_t* rank_of;  // [n_cand] new index of every candidate
    const uint32_t* status;
    uint32_t n;
    uint32_t ntiles;          // tiles of kHashTile rows
    int dim;
    int vec;                  // vtx 16-byte aligned
    int hist_only;            // k_hash_build: histograms only (the first hashed pass stages the vertices)
};

// Cleaned (key words, origin) rows and the digit histograms of the two hashed passes.
template <int D_CT>
__global__ void __launch_bounds__(kBlock) k_hash_build(HashArgs a) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    const int D = D_CT > 0 ? D_CT : a.dim;
    const int W = D + 1;
    __shared__ uint32_t s_hist[kHashPasses * 256];
    for (int i = threadIdx.x; i < kHashPasses * 256; i += kBlock) s_hist[i] = 0u;
    __syncthreads();
    if (*a.status || !hash_mode(a.plan, D)) return;  // uniform
    const uint32_t* repl = a.vtx + static_cast<size_t>(a.idx[0]) * D;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
    const uint64_t start = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    uint32_t rl[kHashPasses] = {};
    auto note = [&](uint32_t h) {
#pragma unroll
        for (int p = 0; p < kHashPasses; ++p) rl_push(rl[p], (h >> (kHashShift0 + 8 * p)) & 255u, s_hist + p * 256);
    };
    uint64_t done = 0;
    if constexpr (D_CT == 3) {
        if (a.vec) {  // 4 rows = 3 x 16 B of vertex words + one flag word -> 4 x 16-byte rows
            uint32_t ref[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) ref[c] = __ldg(repl + c);
            const uint64_t ng = a.n >> 2;
            const uint4* v4 = reinterpret_cast<const uint4*>(a.vtx);
            const uint32_t* f4 = reinterpret_cast<const uint32_t*>(a.flags);
            uint4* r4 = reinterpret_cast<uint4*>(a.rows0);
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
                    note(hash_key<3>(k[j], 3));
                    if (!a.hist_only)
                        __stcs(r4 + 4 * g + j, make_uint4(k[j][0], k[j][1], k[j][2], static_cast<uint32_t>(4 * g + j)));
                }
            }
            done = ng << 2;
        }
    }
    for (uint64_t i = done + start; i < a.n; i += stride) {
        const uint32_t* row = a.flags[i] ? a.vtx + i * D : repl;
        uint32_t k[kHashMaxDim];
        uint32_t* dst = a.rows0 + i * W;
        for (int c = 0; c < D; ++c) {
            k[c] = __ldg(row + c);
            if (!a.hist_only) dst[c] = k[c];
        }
        if (!a.hist_only) dst[D] = static_cast<uint32_t>(i);
        note(hash_key<D_CT>(k, D));
    }
#pragma unroll
    for (int b = 0; b < kHashPasses; ++b)
        if ((rl[b] >> 8) != 0u) atomicAdd(s_hist + b * 256 + (rl[b] & 255u), rl[b] >> 8);
    __syncthreads();
    for (int i = threadIdx.x; i < kHashPasses * 256; i += kBlock)
        if (s_hist[i]) atomicAdd(a.hhist + i, s_hist[i]);
}

__host__ __device__ constexpr int log2_ct(int x) { return x <= 1 ? 0 : 1 + log2_ct(x / 2); }
constexpr int kDedupSlotBits = log2_ct(2 * kHashTile);
constexpr int kDedupSlots = 1 << kDedupSlotBits;  // open-addressing table: load factor <= 1/2
static_assert(kDedupSlots == 2 * kHashTile, "dedup table sized for one tile at load factor 1/2");

__host__ __device__ constexpr size_t hash_dedup_smem(int D) {  // two staging buffers, table, local ids
    return 2 * static_cast<size_t>(kHashTile) * (D + 1) * 4 + kDedupSlots * 4 + kHashTile * 4 + 32;
}

// One tile of hash-grouped rows: its distinct keys (shared-memory table keyed by the
// whole key), one candidate row per distinct key, the group id of every row.
template <int D_CT>
__global__ void __launch_bounds__(kBlock) k_hash_dedup(HashArgs a) {
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    const int D = D_CT > 0 ? D_CT : a.dim;
    const int W = D + 1;
    if (*a.status || !hash_mode(a.plan, D)) return;  // uniform
    uint32_t* s_buf = dyn_smem<uint32_t>();                                  // [2][kHashTile * W] staging
    uint32_t* s_owner = s_buf + 2 * static_cast<size_t>(kHashTile) * W;       // [kDedupSlots] row + 1, 0 = free
    uint32_t* s_lid = s_owner + kDedupSlots;                                  // [kHashTile] local id of a representative
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_lid + kHashTile);         // [2] staging barriers
    __shared__ uint32_t s_warp[kWarps];
    __shared__ uint32_t s_hist[4 * 256];
    __shared__ uint32_t s_base;
    const uint32_t tid = threadIdx.x;
    const uint32_t* grouped = kHashPasses & 1 ? a.rows1 : a.rows0;
    // tiles blockIdx.x, + gridDim.x, ...: the next tile's bulk copy runs while this one is deduplicated
    auto issue = [&](uint32_t tile, uint32_t b) {
        const uint32_t base = tile * static_cast<uint32_t>(kHashTile);
        const uint32_t tn = min(static_cast<uint32_t>(kHashTile), a.n - base);
        stage_tile(s_buf + b * static_cast<size_t>(kHashTile) * W, grouped + static_cast<size_t>(base) * W,
                   tn * W * 4u, s_bar + b);
    };
    if (tid == 0) {
        mbar_init(s_bar, 1);
        mbar_init(s_bar + 1, 1);
        fence_mbar_init();
        if (blockIdx.x < a.ntiles) issue(blockIdx.x, 0u);
    }
    for (uint32_t i = tid; i < 4u * 256u; i += kBlock) s_hist[i] = 0u;
    uint32_t rl[4] = {0u, 0u, 0u, 0u};
    uint32_t it = 0;
    for (uint32_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++it) {  // persistent: a no-op launch is cheap
    const uint32_t base = tile * static_cast<uint32_t>(kHashTile);
    const uint32_t tile_n = min(static_cast<uint32_t>(kHashTile), a.n - base);
    const uint32_t* s_rows = s_buf + (it & 1u) * static_cast<size_t>(kHashTile) * W;
    for (uint32_t i = tid; i < static_cast<uint32_t>(kDedupSlots); i += kBlock) s_owner[i] = 0u;
    // the other buffer was released by the barrier that ended the previous tile
    if (tid == 0 && tile + gridDim.x < a.ntiles) issue(tile + gridDim.x, (it + 1u) & 1u);
    __syncthreads();
    mbar_wait(s_bar + (it & 1u), (it >> 1) & 1u);
    // insert / find every row's key; owner = the row that holds the key's slot.  The first probe
    // of all kHashTileRows rows is issued as a batch (loads, then CASes, then compares: several
    // independent shared-memory round trips in flight per thread instead of one); the rows whose
    // first slot holds another key continue probing one by one.
    uint32_t owner[kHashTileRows], slot[kHashTileRows], o[kHashTileRows];
    auto same_key = [&](uint32_t ra, uint32_t rb) -> bool {
        if constexpr (D_CT == 3) {
            const uint4 x = reinterpret_cast<const uint4*>(s_rows)[ra];
            const uint4 y = reinterpret_cast<const uint4*>(s_rows)[rb];
            return x.x == y.x && x.y == y.y && x.z == y.z;
        } else {
            bool same = true;
            for (int c = 0; c < D; ++c) same = same && s_rows[static_cast<size_t>(ra) * W + c] == s_rows[static_cast<size_t>(rb) * W + c];
            return same;
        }
    };
#pragma unroll
    for (int k = 0; k < kHashTileRows; ++k) {
        const uint32_t r = tid + k * kBlock;
        owner[k] = r;
        slot[k] = r < tile_n ? hash_slot(hash_key<D_CT>(s_rows + static_cast<size_t>(r) * W, D), kDedupSlotBits) : 0u;
    }
#pragma unroll
    for (int k = 0; k < kHashTileRows; ++k) o[k] = tid + k * kBlock < tile_n ? s_owner[slot[k]] : 1u;
#pragma unroll
    for (int k = 0; k < kHashTileRows; ++k) {
        const uint32_t r = tid + k * kBlock;
        if (r < tile_n && o[k] == 0u) {
            o[k] = atomicCAS(s_owner + slot[k], 0u, r + 1u);
            if (o[k] == 0u) o[k] = r + 1u;  // r owns the slot
        }
    }
#pragma unroll
    for (int k = 0; k < kHashTileRows; ++k) {
        const uint32_t r = tid + k * kBlock;
        if (r >= tile_n || o[k] == r + 1u) continue;
        if (same_key(o[k] - 1u, r)) {
            owner[k] = o[k] - 1u;
            continue;
        }
        uint32_t sl = slot[k];
        for (;;) {  // the slot holds another key: linear probing
            sl = (sl + 1u) & (kDedupSlots - 1);
            uint32_t ow = s_owner[sl];
            if (ow == 0u) {
                ow = atomicCAS(s_owner + sl, 0u, r + 1u);
                if (ow == 0u) break;  // r owns the slot
            }
            if (same_key(ow - 1u, r)) {
                owner[k] = ow - 1u;
                break;
            }
        }
    }
    // representatives (owner == self) numbered in row order: flags into s_lid, blocked scan
#pragma unroll
    for (int k = 0; k < kHashTileRows; ++k) {
        const uint32_t r = tid + k * kBlock;
        if (r < tile_n) s_lid[r] = owner[k] == r ? 1u : 0u;
    }
    __syncthreads();
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < kHashTileRows; ++k) {
        const uint32_t r = tid * kHashTileRows + k;
        cnt += r < tile_n ? s_lid[r] : 0u;
    }
    uint32_t total;
    uint32_t run = block_exclusive_scan<kWarps>(cnt, s_warp, total);
    if (tid == 0) s_base = atomicAdd(a.n_cand, total);
    __syncthreads();  // every thread has read its flags before they become local ids
#pragma unroll
    for (int k = 0; k < kHashTileRows; ++k) {
        const uint32_t r = tid * kHashTileRows + k;
        if (r < tile_n && s_lid[r]) s_lid[r] = run++;
    }
    __syncthreads();
    const uint32_t gbase = s_base;
#pragma unroll
    for (int k = 0; k < kHashTileRows; ++k) {
        const uint32_t r = tid + k * kBlock;
        if (r >= tile_n) continue;
        const uint32_t* row = s_rows + static_cast<size_t>(r) * W;
        const uint32_t gid = gbase + s_lid[owner[k]];
        RMX_CHECK_INDEX(gid, a.n);
        RMX_CHECK_INDEX(base + r, a.n);
        __stcs(a.grp_org + base + r, make_uint2(gid, row[D]));
        if (owner[k] == r) {  // the candidate row of this key
            uint32_t* dst = (kHashPasses & 1 ? a.rows0 : a.rows1) + static_cast<size_t>(gid) * W;
            for (int c = 0; c < D; ++c) dst[c] = row[c];
            dst[D] = gid;
            const uint32_t last = row[D - 1];
#pragma unroll
            for (int b = 0; b < 4; ++b) rl_push(rl[b], (last >> (8 * b)) & 255u, s_hist + b * 256);
        }
    }
    __syncthreads();  // the next tile restages s_rows / s_owner / s_lid
    }
#pragma unroll
    for (int b = 0; b < 4; ++b)
        if ((rl[b] >> 8) != 0u) atomicAdd(s_hist + b * 256 + (rl[b] & 255u), rl[b] >> 8);
    __syncthreads();
    for (uint32_t i = tid; i < 4u * 256u; i += kBlock)
        if (s_hist[i]) atomicAdd(a.hist + i, s_hist[i]);
}

// (origin, new index) pairs of the hash-grouped rows, bucketed by the high bits
// of the origin like K3's pairs (k_unique / k_unique_pk), so that k_map_fill's
// stores stay inside an L2-resident window of map (a direct map[origin] store
// per row is a DRAM read-modify-write of a random sector).  The pairs go to the
// row buffer k_map_fill reads in hash mode (both are free by now).
__global__ void __launch_bounds__(kBlock) k_hash_pairs(HashArgs a, uint32_t* fill, int bs) {
    const uint32_t ntiles = (a.n + kPairsTile - 1) / kPairsTile;
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    if (*a.status || !hash_mode(a.plan, a.dim)) return;
    uint2* pairs = reinterpret_cast<uint2*>(a.plan[0] ? a.rows1 : a.rows0);
    __shared__ uint2 s_pairs[kPairsTile];
    __shared__ uint32_t s_bcnt[256], s_bcur[256], s_bglob[256], s_warp[kWarps];
    const uint32_t tid = threadIdx.x;
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {  // persistent: a no-op launch is cheap
    const uint32_t base = tile * static_cast<uint32_t>(kPairsTile);
    const uint32_t tile_n = min(static_cast<uint32_t>(kPairsTile), a.n - base);
    s_bcnt[tid] = 0u;
    __syncthreads();
    uint2 pr[kPairsRows];
#pragma unroll
    for (int k = 0; k < kPairsRows; ++k) {
        const uint32_t r = tid + k * kBlock;
        pr[k] = make_uint2(0u, 0u);
        if (r < tile_n) {
            const uint2 v = __ldcs(a.grp_org + base + r);
            pr[k] = make_uint2(v.y, __ldg(a.rank_of + v.x));
            atomicAdd(s_bcnt + (v.y >> bs), 1u);
        }
    }
    __syncthreads();
    {
        const uint32_t cnt = s_bcnt[tid];
        uint32_t tot;
        const uint32_t start = block_exclusive_scan<kWarps>(cnt, s_warp, tot);
        s_bcur[tid] = start;
        if (cnt) s_bglob[tid] = (tid << bs) + atomicAdd(fill + tid, cnt) - start;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPairsRows; ++k)
        if (tid + k * kBlock < tile_n) s_pairs[atomicAdd(s_bcur + (pr[k].x >> bs), 1u)] = pr[k];
    __syncthreads();
    for (uint32_t q = tid; q < tile_n; q += kBlock) {
        const uint2 p = s_pairs[q];
        RMX_CHECK_INDEX(s_bglob[p.x >> bs] + q, a.n);
        RMX_CHECK_INDEX(p.x, a.n);
        pairs[s_bglob[p.x >> bs] + q] = p;
    }
    __syncthreads();  // the next tile reuses the shared arrays
    }
}

}  // namespace rmx
