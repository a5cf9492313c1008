// rmx_base.cuh -- launch geometry and the device plan layout shared by all kernels.
#pragma once

#include "../../include/remesh_b200.h"
#include "rmx_common.cuh"

namespace rmx {

#ifndef RMX_LB
#define RMX_LB 16  // look-back window (predecessor tiles read per round trip)
#endif

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;

// ---------------------------------------------------------------------------
// Plan layout (uint32 words, lives in the workspace):
//   [0] buffer holding the final sorted rows   [1] executed passes
//   [2] first executed pass                    [3] first pass needs k_first_hist
//   [4 + p]            pass p executes (digit not constant)
//   [4 + P + p]        source buffer of pass p
//   [4 + 2P + p]       next executed pass after p (P = none)
//
// Packed-key section, at word pk_base(P).  When at most 64 key bits vary over
// the (cleaned) vertex set, the varying bits are gathered into one u32/u64
// key -- an order-preserving compaction, since the dropped bits are equal in
// every row -- and the sort runs over (packed key, origin) pairs instead:
//   [0] mode (0 = AoS rows, 1 = packed, 2 = hash: rmx_hash.cuh)
//                                [1] key words KW (1 | 2)   [2] varying bits B
//   [3] packed passes ceil(B/8)  [4] number of runs
//   [5] window mode drops the unused rows in its first pass (no soup mode; in soup mode they keep
//       spread keys and the window kernel skips their origins >= I)
//   [6] window mode (rmx_window.cuh)  [7] window mode's fallback to the full packed path
//   [8 + 4r ..] run r: component, source bit, length, destination bit
//   [8 + 4 kMaxRuns + c] field rank of component c: 0 = none, else
//                        (1 << 31) | (rank bits << 16) | destination bit
// Runs are listed from component D-1 (least significant) to component 0,
// low bits first, so destination bits grow monotonically.
//
// Field ranks (D <= kMaxRankDim): the sign+exponent field (bits 23..31) of a
// float word takes few distinct values in real geometry (coordinates span a few
// binades) but its varying bits are spread over the whole field.  When
// ceil(log2(#distinct fields)) < #varying field bits, the field is replaced in
// the key by its rank among the fields that occur -- monotone and injective on
// them, so order and equality of the words are unchanged -- and the mantissa
// bits keep their runs.  K1a records the occurring fields in a 512-bit set per
// component; pack / unpack build rank / inverse tables from it.
constexpr int kMaxRuns = 64;
constexpr int kMaxPackedPasses = 8;
constexpr int kFieldLo = 23;            // sign + exponent = bits 23..31
constexpr int kFieldValues = 512;
constexpr int kFieldWords = kFieldValues / 32;
constexpr int kMaxRankDim = 4;
__host__ __device__ inline size_t pk_base(int P) { return 4 + 3 * static_cast<size_t>(P); }
__host__ __device__ inline size_t pk_rank_base(int P) { return pk_base(P) + 8 + 4 * kMaxRuns; }

// Value ranks (D <= kMaxRankDim, packed mode): the bits of one component in
// the packed key (its runs and ranked field: contiguous, kMinValueBits ..
// kMaxValueBits wide) are a value cv of that component.  Structured
// coordinates -- lattices, grids, quantised meshes -- take few distinct cv per
// axis although their bits vary widely (C2: 5001 values in 16 bits).  When
// the key gets narrower (fewer 8-bit passes, or u32 instead of u64 keys) cv is
// replaced by its rank among the values that occur: monotone and injective on
// them, so key order and equality are unchanged.  The value sets come from
// k_valueset (a strided sample first, to skip the full pass when even the
// sample needs the full width), the tables from k_value_plan.
//   [0] state: 0 off, 1 full value-set pass wanted, 2 keys carry value ranks
//   [1] candidate components (bit c)
//   [4 + 4c ..] component c: old low bit, old width, new low bit, new width | ranked << 31
constexpr int kMinValueBits = 4;
constexpr int kMaxValueBits = 16;
constexpr int kValueWords = (1 << kMaxValueBits) / 32;
constexpr uint32_t kValueSetBytes = 192 * 1024;  // k_valueset byte maps: sum of 2^w over the candidates
// Hash mode (plan packed-section word 0 == 2, rmx_hash.cuh): keys wider than 64 bits are
// deduplicated by a 32-bit hash first and only the distinct rows are sorted exactly.
constexpr int kHashPasses = 3;       // hashed passes: the top 24 bits of the key hash (~9 rows per
                                     // bucket in C2s, so a dedup tile splits few keys)
constexpr int kHashShift0 = 8 * (4 - kHashPasses);  // the first hashed digit's bit offset
#ifndef RMX_HASH_ROWS
#define RMX_HASH_ROWS 4
#endif
constexpr int kHashTileRows = RMX_HASH_ROWS;  // rows per thread in the hash tile kernels
constexpr int kHashTile = kBlock * kHashTileRows;    // dedup tile
constexpr int kPairsRows = 8;                        // k_hash_pairs: rows per thread
constexpr int kPairsTile = kBlock * kPairsRows;
constexpr int kHashMaxDim = 8;       // wider rows take the AoS path

__host__ __device__ inline size_t pk_value_base(int P) { return pk_rank_base(P) + RMX_MAX_DIM; }
__host__ __device__ inline size_t plan_words(int P) { return pk_value_base(P) + 4 + 4 * kMaxRankDim; }

}  // namespace rmx
