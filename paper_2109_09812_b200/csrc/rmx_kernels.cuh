// rmx_kernels.cuh -- the sm_100a kernels of the re-indexing pipeline.
//
//   K1   k_mark         isUsed scatter over the index buffer + range check
//                       (reference mark_used pipeline.py:41-51, require_valid mesh.py:103-105)
//   K1b  k_build_rows   unused -> replacement, AoS (key words, origin) rows,
//                       per-component varying-bit masks, component D-1 digit
//                       histograms (overwrite_unused pipeline.py:54-63,
//                       fill_sequence primitives.py:16-20)
//   plan k_plan         digit-pass skipping, ping-pong schedule, pass chaining
//   hist k_first_hist   histogram of the first executed pass if K1b lacks it
//   K2   k_sort_pass    one onesweep LSD pass: double-buffered TMA-bulk tile
//                       staging, warp multi-split ranking, windowed decoupled
//                       look-back, smem reorder, next pass's histogram
//                       (bitwise_sort_order / key_value_sort primitives.py:23-40)
//   K3   k_unique       adjacent-compare head flags + decoupled look-back scan,
//                       unique-row compaction, bucketed (org, new_idx) pairs
//                       (pipeline.py:72-113, primitives.py:43-69)
//   K3b  k_map_fill     map[org] = new_idx from the bucket-major pairs
//   K4   k_remap        out_idx = map[idx] (remap_elements pipeline.py:116-130)
//   hash k_hash_*       keys wider than 64 bits: dedup by hash, exact sort of the
//                       distinct rows only (rmx_hash.cuh)
//   small k_small       the whole pipeline in one CTA for small meshes (rmx_small.cuh)
//   merge k_merge_path  sorted-run merge + unique of the multi-GPU exchange (rmx_merge.cuh)
//   gen  k_gen_lattice  synthetic bench input (oracle/lattice.py recipe)
//
// Data layout in HBM: a row is W = D+1 uint32 words -- the D key words of the
// (cleaned) vertex followed by its original index.  Rows are AoS so one tile
// of rows is one contiguous byte range, moved into shared memory with a
// single cp.async.bulk.  Key order is the reference's: raw unsigned words,
// component 0 most significant, so LSD pass p sorts byte (p % 4) of
// component D-1-p/4, pass 0 first.
#pragma once

#include "rmx_prep.cuh"
#include "rmx_sort.cuh"
#include "rmx_unique.cuh"
#include "rmx_hash.cuh"
#include "rmx_packed.cuh"
#include "rmx_window.cuh"
#include "rmx_gen.cuh"
#include "rmx_steps.cuh"
#include "rmx_small.cuh"
#include "rmx_merge.cuh"
