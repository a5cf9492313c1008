// rmx_sort.cuh -- K2 onesweep LSD pass over AoS (key words, origin) rows.
#pragma once

#include "rmx_base.cuh"
#include "rmx_hashfn.cuh"

namespace rmx {

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
    int rank_force;  // -1 = choose per pass; else kRankMatch / kRankBallot / kRankAtomic
    const uint32_t* n_cand;  // hash mode: the rows are the n_cand candidate rows
    // hash mode, first hashed pass over D = 3 vertices (RAW): the tile is staged straight from the
    // vertex words and the used flags, cleaned and given its origin on the way out
    const uint32_t* raw_vtx;
    const uint8_t* raw_flags;
    const uint32_t* raw_idx;
    // RAW in soup mode (rmx_packed.cuh k_soup_decide): used row o gets the origin "used rows before
    // o" (its index position), unused row o I + "unused rows before o"; soup_prefix: used rows
    // before every tile
    const uint32_t* soup;
    const uint32_t* soup_prefix;
};

template <int W_CT, int IPT>
struct SortTraits {
    static constexpr int kTile = kBlock * IPT;
    static __host__ __device__ size_t smem_bytes(int W) {
        return static_cast<size_t>(kTile) * W * 4 + static_cast<size_t>(kTile) * 2 +
               (2 * kWarps * 256 + 256 * 3 + kWarps + 8) * 4 + 16;
    }
};

template <int W_CT>
__device__ __forceinline__ uint32_t pick_word(const uint4& v, int comp) {
    return comp == 0 ? v.x : (comp == 1 ? v.y : v.z);
}

// D = 3, 4 rows: 5120 / 4096-row tiles at 2 CTAs per SM (measured against 3072 / 2560 rows at 3:
// scrambled C2 22.0 -> 20.6 ms, C3 18.5 -> 17.3 ms, tools/aos_probe.py); other widths 3 CTAs per SM
template <int W_CT>
struct SortMinBlocks { static constexpr int v = (W_CT == 4 || W_CT == 5) ? 2 : 3; };

// HASHED (hash mode, rmx_hash.cuh): the digit is byte (4 - kHashPasses + pass) of hash_key(row) --
// kHashPasses passes group the whole vertex set by the top bits of its key hash (a.hist / a.counters
// are then the hashed passes' own arrays, rows0 -> rows1 -> ...).
template <int W_CT, int IPT, bool HASHED = false, bool RAW = false, bool SOUP = false>
__global__ void __launch_bounds__(kBlock, SortMinBlocks<W_CT>::v) k_sort_pass(SortArgs a) {
    static_assert(!RAW || (HASHED && W_CT == 4), "raw staging: the first hashed pass over float3 vertices");
    static_assert(!SOUP || RAW, "soup origins are made by the raw pass");
    pdl_enter();  // programmatic dependent launch: wait for the previous kernel
    using T = SortTraits<W_CT, IPT>;
    constexpr int TILE = T::kTile;
    const int W = W_CT > 0 ? W_CT : a.dim + 1;
    const int D = W - 1;
    const int P = 4 * a.dim;
    if (*a.status) return;
    const uint32_t* plan = a.plan;
    const bool hash = plan[pk_base(P)] == 2u;
    if (HASHED ? !hash : plan[4 + a.pass] == 0u) return;  // constant digit (or not this mode): nothing moves
    if constexpr (RAW) {  // the soup variant and the plain one: the one that matches runs
        if ((a.soup && *a.soup != 0u) != SOUP) return;
    }
    // AoS mode sorts the whole vertex set, hash mode its n_cand candidate rows (HASHED: all rows)
    const uint32_t n = (hash && !HASHED) ? *a.n_cand : a.n;
    const uint32_t ntiles = (n + static_cast<uint32_t>(TILE) - 1u) / static_cast<uint32_t>(TILE);
    const uint32_t src = HASHED ? static_cast<uint32_t>(a.pass & 1) : plan[4 + P + a.pass];
    const uint32_t* __restrict__ in = src ? a.rows1 : a.rows0;
    uint32_t* __restrict__ out = src ? a.rows0 : a.rows1;
    const int comp = a.dim - 1 - (a.pass >> 2);
    const int shift = HASHED ? kHashShift0 + 8 * a.pass : 8 * (a.pass & 3);
    const uint32_t epoch = HASHED ? 200u + static_cast<uint32_t>(a.pass) : static_cast<uint32_t>(a.pass) + 1u;
    const int nxt = HASHED ? P : static_cast<int>(plan[4 + 2 * P + a.pass]);
    // passes 0..3 are counted by K1b; later ones by the pass before them
    const bool count_next = nxt < P && nxt >= 4;
    const int ncomp = count_next ? a.dim - 1 - (nxt >> 2) : 0;
    const int nshift = 8 * (nxt & 3);
    uint32_t* ctr = a.counters + a.pass;
    // the digit of a staged row
    auto digit_of = [&](const uint32_t* row) -> uint32_t {
        if constexpr (HASHED) return (hash_key<W_CT - 1>(row, D) >> shift) & 255u;
        else return (row[comp] >> shift) & 255u;
    };
    uint32_t repl[3] = {0u, 0u, 0u};  // RAW: the replacement row (pipeline.py:148)
    if constexpr (RAW) {
        const uint32_t r0 = a.raw_idx[0];
#pragma unroll
        for (int c = 0; c < 3; ++c) repl[c] = __ldg(a.raw_vtx + static_cast<size_t>(r0) * 3 + c);
    }

    uint32_t* smem = dyn_smem<uint32_t>();
    const size_t tw = static_cast<size_t>(TILE) * W;
    uint32_t* s_rows = smem;                          // [TILE * W]
    uint32_t* s_whist = smem + tw;                    // [warp][256] digit counters
    uint32_t* s_wmask = s_whist + kWarps * 256;       // [warp][256] peer masks (zero between rounds)
    uint32_t* s_offs = s_wmask + kWarps * 256;        // global exclusive digit starts
    uint32_t* s_gdst = s_offs + 256;                  // global row of tile slot 0, per digit
    uint32_t* s_hnext = s_gdst + 256;                 // histogram of the next executed pass
    uint32_t* s_warp = s_hnext + 256;
    uint32_t* s_misc = s_warp + kWarps;
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_misc + 8);
    uint16_t* s_src = reinterpret_cast<uint16_t*>(s_bar + 2);  // slot -> row of the staged tile

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    if (tid == 0) {
        mbar_init(s_bar, 1);
        fence_mbar_init();
    }
    const uint32_t h = a.hist[a.pass * 256 + tid];
    {
        uint32_t tot;
        s_offs[tid] = block_exclusive_scan<kWarps>(h, s_warp, tot);
        s_hnext[tid] = 0u;
        for (int i = tid; i < kWarps * 256; i += kBlock) s_wmask[i] = 0u;
    }
    const int rank_mode = choose_rank(a.hist[a.pass * 256 + tid], a.rank_force);
    for (uint32_t it = 0;; ++it) {
        if (tid == 0) {
            const uint32_t t = atomicAdd(ctr, 1u);
            s_misc[0] = t;
            if (t < ntiles) {
                const uint32_t tn = min(static_cast<uint32_t>(TILE), n - t * static_cast<uint32_t>(TILE));
                if constexpr (RAW)  // vertex words [TILE * 3] then flags [TILE] (sizes round up to 16 B)
                    stage_tile2(s_rows, a.raw_vtx + static_cast<size_t>(t) * TILE * 3, tn * 12u, s_rows + TILE * 3,
                                a.raw_flags + static_cast<size_t>(t) * TILE, tn, s_bar);
                else
                    stage_tile(s_rows, in + static_cast<size_t>(t) * TILE * W, tn * W * 4u, s_bar);
            }
        }
        for (int i = tid; i < kWarps * 256; i += kBlock) s_whist[i] = 0u;
        __syncthreads();
        const uint32_t tile = s_misc[0];
        if (tile >= ntiles) break;
        const uint32_t tile_n = min(static_cast<uint32_t>(TILE), n - tile * static_cast<uint32_t>(TILE));
        mbar_wait(s_bar, it & 1u);
        // RAW, soup mode: a used mask per 32 rows (in the staging buffer's spare bytes past the
        // flags; made by the digit loop), the used rows before each 32 (in the digit scan)
        uint32_t* s_umask = s_rows + TILE * 13 / 4;  // [TILE / 32] masks, then [TILE / 32] prefixes
        uint32_t soup_n = 0, soup_base = 0;
        if constexpr (SOUP) {
            soup_n = *a.soup;
            soup_base = a.soup_prefix[tile];
        }

        // ---- digits (+ next pass's histogram), stable warp ranks
        uint32_t pk[IPT];
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
            uint32_t d = 256u;
            if (p < tile_n) {
                uint32_t key, nkey = 0;
                if constexpr (RAW) {
                    key = 0u;
                    const uint8_t* s_fl = reinterpret_cast<const uint8_t*>(s_rows + TILE * 3);
                    d = digit_of(s_fl[p] ? s_rows + static_cast<size_t>(p) * 3 : repl);
                } else if constexpr (HASHED) {
                    key = 0u;
                    d = digit_of(s_rows + static_cast<size_t>(p) * W);
                } else if constexpr (W_CT == 4) {
                    const uint4 v = reinterpret_cast<const uint4*>(s_rows)[p];
                    key = pick_word<4>(v, comp);
                    if (count_next) nkey = pick_word<4>(v, ncomp);
                    d = (key >> shift) & 255u;
                } else {
                    key = s_rows[static_cast<size_t>(p) * W + comp];
                    if (count_next) nkey = s_rows[static_cast<size_t>(p) * W + ncomp];
                    d = (key >> shift) & 255u;
                }
                if (count_next) atomicAdd(s_hnext + ((nkey >> nshift) & 255u), 1u);
            }
            pk[r] = d;
            if constexpr (SOUP) {  // rows 32 (warp * IPT + r) .. +31: the used mask
                const uint8_t* s_fl = reinterpret_cast<const uint8_t*>(s_rows + TILE * 3);
                const uint32_t bal = __ballot_sync(kFull, p < tile_n && s_fl[p] != 0);
                if (lane == 0u) s_umask[warp * IPT + r] = bal;
            }
        }
        warp_rank<IPT>(pk, s_whist + warp * 256, s_wmask + warp * 256, rank_mode, tile_n < static_cast<uint32_t>(TILE));
        __syncthreads();

        // ---- per digit: count, publish aggregate, tile-local start
        const uint32_t d = tid;
        uint32_t cnt = 0, start;
        {
            uint32_t wc[kWarps];
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                wc[w] = s_whist[w * 256 + hsw(d)];
                cnt += wc[w];
            }
            st_relaxed(a.desc + static_cast<size_t>(tile) * 256 + d,
                       pack_desc(epoch, tile == 0 ? kPrefix : kAggregate, cnt));
            uint32_t tot;
            if constexpr (SOUP) {  // + the used rows before every 32 rows, in the high half
                constexpr uint32_t kChunks = static_cast<uint32_t>(TILE) / 32u;
                static_assert(TILE < 65536 && kChunks <= kBlock, "packed scan of digit counts and used counts");
                const uint32_t uc = tid < kChunks ? __popc(s_umask[tid]) : 0u;
                const uint32_t both = block_exclusive_scan<kWarps>(cnt | (uc << 16), s_warp, tot);
                start = both & 0xFFFFu;
                if (tid < kChunks) s_umask[kChunks + tid] = both >> 16;
            } else {
                start = block_exclusive_scan<kWarps>(cnt, s_warp, tot);
            }
            uint32_t run = start;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                s_whist[w * 256 + hsw(d)] = run;
                run += wc[w];
            }
        }
        __syncthreads();
        // ---- reorder (local) while predecessors finish publishing
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
            const uint32_t p = warp * (32u * IPT) + r * 32u + lane;
            if (p < tile_n) s_src[s_whist[warp * 256 + (pk[r] >> 16)] + (pk[r] & 0xFFFFu)] = static_cast<uint16_t>(p);
        }
        // ---- look-back: global start of this tile's run of digit d
        {
            uint32_t excl = 0;
            if (tile > 0) {
                excl = lookback_digit<RMX_LB>(a.desc, tile, d, epoch);
                st_relaxed(a.desc + static_cast<size_t>(tile) * 256 + d, pack_desc(epoch, kPrefix, excl + cnt));
            }
            s_gdst[d] = s_offs[d] + excl - start;  // mod 2^32; + tile slot gives the global row
        }
        __syncthreads();

        // ---- coalesced write-out: consecutive slots of one digit are consecutive rows
        if constexpr (W_CT == 4) {
            const uint4* s4 = reinterpret_cast<const uint4*>(s_rows);
            uint4* o4 = reinterpret_cast<uint4*>(out);
            constexpr int U = 4;
            for (uint32_t q0 = tid; q0 < tile_n; q0 += U * kBlock) {
                uint4 v[U];
                uint32_t dst[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t q = q0 + u * kBlock;
                    if (q < tile_n) {
                        if constexpr (RAW) {  // cleaned row + its origin
                            const uint32_t p = s_src[q];
                            const uint8_t* s_fl = reinterpret_cast<const uint8_t*>(s_rows + TILE * 3);
                            const uint32_t* r = s_fl[p] ? s_rows + static_cast<size_t>(p) * 3 : repl;
                            uint32_t org = tile * static_cast<uint32_t>(TILE) + p;
                            if constexpr (SOUP) {
                                const uint32_t before = soup_base + s_umask[TILE / 32 + (p >> 5)] +
                                                        __popc(s_umask[p >> 5] & ((1u << (p & 31u)) - 1u));
                                org = s_fl[p] ? before : soup_n + org - before;
                            }
                            v[u] = make_uint4(r[0], r[1], r[2], org);
                        } else {
                            v[u] = s4[s_src[q]];
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t q = q0 + u * kBlock;
                    if (q < tile_n) {
                        if constexpr (HASHED) {  // the digit again (a cached digit per slot costs a CTA/SM)
                            const uint32_t row[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
                            dst[u] = s_gdst[digit_of(row)] + q;
                        } else {
                            dst[u] = s_gdst[(pick_word<4>(v[u], comp) >> shift) & 255u] + q;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t q = q0 + u * kBlock;
                    if (q < tile_n) {
                        RMX_CHECK_INDEX(dst[u], n);
                        o4[dst[u]] = v[u];
                    }
                }
            }
        } else {
            const uint32_t nw = tile_n * W;
            for (uint32_t q = tid; q < nw; q += kBlock) {
                const uint32_t slot = q / W;
                const uint32_t c = q - slot * W;
                const size_t p = s_src[slot];
                const uint32_t dd = digit_of(s_rows + p * W);
                RMX_CHECK_INDEX(s_gdst[dd] + slot, n);
                out[static_cast<size_t>(s_gdst[dd] + slot) * W + c] = s_rows[p * W + c];
            }
        }
        __syncthreads();
    }
    if (count_next && s_hnext[tid]) atomicAdd(a.hist + nxt * 256 + tid, s_hnext[tid]);
}

}  // namespace rmx
