/*
 * remesh_b200.h -- C-ABI of the B200-native re-indexing hot path.
 *
 * The reference (remeshx 0.1.0, /root/reference/pkg) is a pure Python/numpy
 * package with no FFI; its operator API is the module-level Python function
 *
 *     reindex(mesh: Mesh) -> tuple[Mesh, ReindexScratch]      pipeline.py:133-157
 *
 * re-exported at __init__.py:12-15 and bound by name in ops.py:7, cli.py:17,
 * bench.py:19 and testing.py:18.  This header is the native boundary that
 * the Python drop-in (paper_2109_09812_b200.pipeline.reindex) calls through
 * ctypes.  Plain pointers and sizes only; no torch types.  All pointers
 * except the host-side `rmx_scratch` struct itself are DEVICE pointers; every
 * call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy default)
 * and never allocates: the caller owns every buffer, including the
 * workspace sized by rmx_workspace_bytes() (256-byte aligned, as
 * cudaMalloc and torch allocations are; RMX_EINVAL otherwise).
 *
 * Vertex data is handled exclusively as uint32 words (the reference's
 * `vertex_bits`, mesh.py:91-94): ordering is raw unsigned bit order,
 * component 0 most significant (primitives.py:23-27); equality is bitwise.
 */
#ifndef REMESH_B200_H
#define REMESH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes */
#define RMX_OK        0
#define RMX_EINVAL    1   /* bad shape/pointer/size (reference: MeshError, mesh.py:55-60) */
#define RMX_ERANGE    2   /* n_vertices >= 2^32 (reference: MeshError, mesh.py:59-60)    */
#define RMX_ECUDA     3   /* a CUDA runtime call failed                                 */
#define RMX_ENOSPC    4   /* workspace smaller than rmx_workspace_bytes()               */

/* bits of the device status word written by the pipeline */
#define RMX_STATUS_INDEX_OUT_OF_RANGE 1u   /* reference: InvalidMeshError, mesh.py:103-105 */
#define RMX_STATUS_LEAN_UNSUPPORTED 2u     /* rmx_reindex_lean: more than 64 key bits vary */

/* largest vertex dimension the CUDA path accepts (reference: unbounded) */
#define RMX_MAX_DIM 32

/* Optional intermediates of one run (reference ReindexScratch, pipeline.py:24-38).
 * Any field may be NULL; all are device pointers of length n_vertices. */
typedef struct rmx_scratch {
    uint8_t*  is_used;   /* bool per input vertex          (pipeline.py:41-51)   */
    uint32_t* org_id;    /* origin of each sorted slot      (pipeline.py:66-69)   */
    uint8_t*  nodup;     /* first-occurrence flag per slot  (pipeline.py:72-83)   */
    uint32_t* new_idx;   /* compacted destination per slot  (pipeline.py:86-94)   */
    uint32_t* perm;      /* inverse of org_id               (pipeline.py:103-113) */
} rmx_scratch;

/* Library identification. */
const char* rmx_version(void);
const char* rmx_strerror(int code);

/* Bytes of device workspace rmx_reindex needs for this problem size
 * (the "two copies of vertex and index data" of SPEC.md are the caller's
 * in/out buffers; this is the sort ping-pong, flags, map and look-back state). */
size_t rmx_workspace_bytes(uint64_t n_vertices, uint32_t dim,
                           uint64_t n_elements, uint32_t arity);

/*
 * Full re-indexing pipeline.  Replaces remeshx.reindex (pipeline.py:133-157)
 * and every step it calls:
 *   require_valid    mesh.py:103-105       -> status bit, checked by caller
 *   mark_used        pipeline.py:41-51     -> K1  mark scatter
 *   overwrite_unused pipeline.py:54-63     -> K1b replace + row build + digit histograms
 *   compute_sort_permutation / key_value_sort / bitwise_sort_order
 *                    pipeline.py:66-69, primitives.py:23-40 -> K2 onesweep LSD passes
 *   flag_first_occurrences, compute_new_indices, compact_vertices, invert_permutation
 *                    pipeline.py:72-113    -> K3 head flag + look-back scan + map + gather
 *   remap_elements   pipeline.py:116-130   -> K4 remap
 *
 * vtx_bits     [n_vertices * dim]   input vertex words (row-major)
 * idx          [n_elements * arity] input element indices (row-major)
 * out_vtx_bits [n_vertices * dim]   capacity; the first *d_new_count rows are the result
 * out_idx      [n_elements * arity] remapped indices
 * d_new_count  device uint64: number of output vertices
 * d_status     device uint32: RMX_STATUS_* bits (non-zero => outputs are undefined)
 * scratch      NULL, or host struct of device pointers to fill
 * stream       cudaStream_t
 * Zero elements: writes new_count = 0 and is_used = all false, like pipeline.py:142-146.
 */
int rmx_reindex(const uint32_t* vtx_bits, uint64_t n_vertices, uint32_t dim,
                const uint32_t* idx, uint64_t n_elements, uint32_t arity,
                uint32_t* out_vtx_bits, uint32_t* out_idx,
                uint64_t* d_new_count, uint32_t* d_status,
                void* workspace, size_t workspace_bytes,
                const rmx_scratch* scratch, void* stream);

/* Same as rmx_reindex, additionally recording `events[k]` (cudaEvent_t
 * handles created by the caller) on `stream` after the k-th stage boundary,
 * k = 0 .. min(n_events, rmx_stage_count(dim)) - 1.  Stage 0 is the start.
 * Used by bench.py to time each kernel live inside the timed region. */
int rmx_reindex_profiled(const uint32_t* vtx_bits, uint64_t n_vertices, uint32_t dim,
                         const uint32_t* idx, uint64_t n_elements, uint32_t arity,
                         uint32_t* out_vtx_bits, uint32_t* out_idx,
                         uint64_t* d_new_count, uint32_t* d_status,
                         void* workspace, size_t workspace_bytes,
                         const rmx_scratch* scratch, void* stream,
                         void* const* events, int n_events);

/*
 * Graph launch path: the whole rmx_reindex call for these exact buffers and
 * sizes, captured once into a CUDA graph.  The sections that only some inputs
 * need (AoS rows vs packed keys, every sort pass) are IF conditional nodes the
 * plan kernel switches on the device, so no kernel of a path not taken is
 * launched.  Replaces repeated rmx_reindex calls on fixed buffers (the
 * reference's bench loop, pkg/src/remeshx/bench.py:71-94, calls reindex on the
 * same mesh repeatedly); results are identical to rmx_reindex.
 *   rmx_graph_create   builds and instantiates (host-side, no stream work);
 *   rmx_graph_launch   enqueues one re-index on `stream`;
 *   rmx_graph_destroy  frees it.
 */
typedef struct rmx_graph rmx_graph;
int rmx_graph_create(const uint32_t* vtx_bits, uint64_t n_vertices, uint32_t dim,
                     const uint32_t* idx, uint64_t n_elements, uint32_t arity,
                     uint32_t* out_vtx_bits, uint32_t* out_idx,
                     uint64_t* d_new_count, uint32_t* d_status,
                     void* workspace, size_t workspace_bytes,
                     const rmx_scratch* scratch, rmx_graph** out);
int rmx_graph_launch(rmx_graph* graph, void* stream);
void rmx_graph_destroy(rmx_graph* graph);

/* Memory-lean re-index (opt-in, no reference counterpart:
 * it breaks the pure-function contract of pipeline.py:133-157 on purpose).
 * The caller's vertex buffer is OVERWRITTEN -- after the keys are built it is
 * the second sort buffer -- and the unique rows (U x dim words) are left in the
 * final sort buffer: *d_where = 0 -> the workspace at offset
 * rmx_lean_result_offset(), 1 -> the vertex buffer itself.  Keys must pack into
 * 64 bits (lattice-like and quantised data); otherwise RMX_STATUS_LEAN_UNSUPPORTED
 * is set in *d_status and nothing is produced.  dim >= 3, n_vertices even and
 * above the one-CTA size, no scratch.  Workspace about 40 B per vertex (C5:
 * 3.15B vertices re-indexed on one 180 GB GPU). */
size_t rmx_lean_workspace_bytes(uint64_t n_vertices, uint32_t dim, uint64_t n_elements, uint32_t arity);
size_t rmx_lean_result_offset(uint64_t n_vertices, uint32_t dim);
int rmx_reindex_lean(uint32_t* vtx_bits, uint64_t n_vertices, uint32_t dim, const uint32_t* idx,
                     uint64_t n_elements, uint32_t arity, uint32_t* out_idx, uint64_t* d_new_count,
                     uint32_t* d_status, uint32_t* d_where, void* workspace, size_t workspace_bytes,
                     void* stream);

/* Number of stage-boundary events rmx_reindex_profiled records for `dim`, and
 * the name of the kernel that runs between event k-1 and event k. */
int rmx_stage_count(uint32_t dim);
const char* rmx_stage_name(uint32_t dim, int k);

/* Kernels one rmx_reindex call launches (n_elements > 0).  The plan is made on
 * the device, so the kernels of the path not taken (AoS rows vs packed keys,
 * constant digits) are still launched and return at once. */
int rmx_kernel_launches(uint32_t dim);

/* Kernels the re-indexing pipeline has launched in this process so far (all
 * calls, all threads): the difference around a region counts its launches. */
unsigned long long rmx_kernel_launches_total(void);

/* Checked builds only (-DRMX_CHECKED): scattered stores whose index was past its array, summed over
 * the process (synchronises the device); RMX_EINVAL in ordinary builds. */
int rmx_debug_oob_count(unsigned long long* out);

/* Sort plan of the last call that used `workspace` (host-side diagnostic; it
 * reads the device plan, so it synchronises `stream`).  Digit passes whose
 * 8-bit digit is constant over all keys are skipped; when at most 64 key bits
 * vary, the varying bits are packed into one u32/u64 key (order-preserving).
 * rmx_last_executed_passes returns the executed sort passes;
 * rmx_plan_info fills info[4] = {packed, key words, varying bits, passes};
 * rmx_plan_key_info fills info[4] = {field-ranked components (bit mask),
 * value-ranked components (bit mask), key bits before value ranks, key bits}
 * (zeros unless packed). */
int rmx_last_executed_passes(void* workspace, uint64_t n_vertices, uint32_t dim, void* stream);
int rmx_plan_info(void* workspace, uint64_t n_vertices, uint32_t dim, void* stream, uint32_t* info);
int rmx_plan_key_info(void* workspace, uint64_t n_vertices, uint32_t dim, void* stream, uint32_t* info);
/* Diagnostic of the value-rank guess (D <= 4): info[4] = {key bits of the plan guessed from the
 * sample, value sets judged worth collecting (0/1), candidate components, full-pass check state
 * (bit 0 checked, bit 1 a row fell outside the sample; bit 8 the plan was speculative -- the
 * sample halves saw the same value sets, no full value-set pass --, bit 9 k_pack's check of the
 * speculative plan failed and the skipped path ran)}. */
int rmx_plan_guess_info(void* workspace, uint64_t n_vertices, uint32_t dim, void* stream, uint32_t* info);

/* Soup mode of the last call that used `workspace` (synchronises `stream`): info[2] = {the index
 * count I when soup mode ran -- strictly increasing indices and a packed plan: used vertex o is
 * sorted with its index position as origin, so the map fill writes the output indices and no
 * remap runs --, else 0; 1 if the indices were strictly increasing}. */
int rmx_soup_info(void* workspace, uint64_t n_vertices, uint32_t dim, void* stream, uint32_t* info);

/* Window mode of the last call that used `workspace` (u32 packed keys of 25..32 bits sorted by
 * their top 16 bits, per-window presence bitmaps; synchronises `stream`): info[4] = {bit 0 window
 * mode decided, bit 1 its fallback ran; rows of the window passes (soup mode: all slots, else the
 * used rows); non-empty windows; rows of the largest window}.  Diagnostic; no reference
 * counterpart. */
int rmx_window_info(void* workspace, uint64_t n_vertices, uint32_t dim, void* stream, uint32_t* info);

/* Hash mode of the last call that used `workspace` (keys wider than 64 bits, no
 * scratch requested; synchronises `stream`): info[4] = {ran in hash mode,
 * candidate rows (distinct keys per dedup tile), executed AoS passes over the
 * candidates, rows per dedup tile}. */
int rmx_hash_info(void* workspace, uint64_t n_vertices, uint32_t dim, void* stream, uint32_t* info);

/* Tuning diagnostic: look-back statistics {windows, spins, look-backs, 0} of
 * the AoS sort passes when built with -DRMX_PHASES (otherwise zeros; returns 0). */
int rmx_debug_phase_cycles(unsigned long long* out, int n, int reset);

/*
 * Steps of the multi-GPU path (paper_2109_09812_b200/dist.py).
 * rmx_gather_u32: out[i] = table[idx[i]] -- the remap of remap_elements
 *   (pipeline.py:116-130) with a caller-supplied table; an index >= n_table
 *   sets RMX_STATUS_INDEX_OUT_OF_RANGE in *d_status and leaves out[i] unwritten.
 * rmx_lower_bound_rows: for each query row, the first position in the sorted
 *   rows[0..n) whose row is >= the query in the reference's bitwise order
 *   (component 0 most significant, raw unsigned words; primitives.py:23-27).
 */
int rmx_gather_u32(const uint32_t* table, uint64_t n_table, const uint32_t* idx, uint64_t n,
                   uint32_t* out, uint32_t* d_status, void* stream);
int rmx_lower_bound_rows(const uint32_t* rows, uint64_t n, uint32_t dim, const uint32_t* queries,
                         uint64_t n_queries, uint64_t* out_positions, void* stream);

/*
 * Synthetic lattice soups of BASELINE.md section 3 (bench input generator;
 * not part of the reference interface).  kind 0 = triangles (dim 3, arity 3,
 * cells nx*ny), kind 1 = Kuhn tetrahedra (dim 4, arity 4, cells nx*ny*nz).
 * Writes n_vertices*dim words to out_vtx_bits and n_elem_take*arity indices
 * to out_idx, bit-identical to oracle/lattice.py:lattice_soup.
 * rmx_lattice_sizes reports (n_elements_total, n_vertices_for_take).
 */
int rmx_lattice_sizes(int kind, uint32_t nx, uint32_t ny, uint32_t nz,
                      uint64_t n_elem_take, uint64_t* n_elements, uint64_t* n_vertices);
int rmx_gen_lattice_soup(int kind, uint32_t nx, uint32_t ny, uint32_t nz, uint64_t seed,
                         uint64_t n_elem_take, uint32_t* out_vtx_bits, uint32_t* out_idx,
                         void* stream);
/* Elements [e_begin, e_end) of the same soup with the vertex slots they own
 * (up to the next element), indices relative to the first written slot: one
 * rank's shard of a soup partitioned across GPUs.  Slot count of a range =
 * rmx_lattice_sizes(e_end) - rmx_lattice_sizes(e_begin). */
int rmx_gen_lattice_soup_range(int kind, uint32_t nx, uint32_t ny, uint32_t nz, uint64_t seed,
                               uint64_t e_begin, uint64_t e_end, uint32_t* out_vtx_bits,
                               uint32_t* out_idx, void* stream);

/*
 * subset (reference pkg/src/remeshx/ops.py:59-68) on the device: the elements
 * e with keep[e] != 0 (u8 per element, device), in order, into out_idx
 * (capacity n_elements x arity); their number to *d_kept (device).
 */
size_t rmx_select_workspace_bytes(uint64_t n_elements);
int rmx_select_elements(const uint32_t* idx, uint64_t n_elements, uint32_t arity, const uint8_t* keep,
                        uint32_t* out_idx, uint64_t* d_kept, void* workspace, size_t workspace_bytes,
                        void* stream);

/*
 * merge (reference pkg/src/remeshx/ops.py:29-34) on the device: out[i] =
 * idx[i] + offset (mod 2^32), the index array of one piece shifted by the
 * vertex count of the pieces before it in the concatenation.
 */
int rmx_offset_indices(const uint32_t* idx, uint64_t n, uint32_t offset, uint32_t* out, void* stream);

/*
 * Distributed exchange over peer memory:
 * rows [bounds[g], bounds[g+1]) of src (n rows of `words` u32, sorted by
 * destination) are stored into the buffer at dst_ptrs[g] (a peer GPU's
 * symmetric receive buffer, reached over NVLink) starting at row dst_off[g].
 * bounds (groups+1 entries), dst_ptrs and dst_off (groups entries) are
 * DEVICE arrays.  Replaces the send staging + NCCL all-to-all of
 * dist.py's exchange; the caller orders it with a barrier on the receivers.
 */
int rmx_scatter_rows(const uint32_t* src, uint64_t n, uint32_t words, const uint64_t* bounds, uint32_t groups,
                     const uint64_t* dst_ptrs, const uint64_t* dst_off, void* stream);

/*
 * Multi-GPU step 4 (dist.py): keys (n_rows x key_words u32) are n_runs runs,
 * run r = rows [run_starts[r], run_starts[r+1]) (host array), each sorted
 * lexicographically (word 0 most significant) and duplicate-free.  Writes the
 * sorted unique keys to out_keys (capacity n_rows x key_words), the index in
 * out_keys of every input row to rank_of[n_rows], and their count to
 * *d_new_count (device).  Pairwise merge-path rounds, then one compaction.
 * key_words <= 8.
 */
size_t rmx_merge_workspace_bytes(uint64_t n_rows, uint32_t key_words);
int rmx_merge_unique_runs(const uint32_t* keys, uint64_t n_rows, uint32_t key_words, const uint64_t* run_starts,
                          uint32_t n_runs, uint32_t* out_keys, uint32_t* rank_of, uint64_t* d_new_count,
                          void* workspace, size_t workspace_bytes, void* stream);

/*
 * Welded (indexed) tile of the C4 merge workload:
 * the triangulated n x n quad grid whose lattice rows start at row0, every
 * point stored once, 5 % unused rows; points and triangles row-major, or
 * with shuffle != 0 at seeded positions / in seeded order (the random-access
 * case); bit-identical to oracle/lattice.py:welded_tile.
 */
int rmx_welded_tile_sizes(uint32_t n, uint64_t* n_vertices, uint64_t* n_elements);
int rmx_gen_welded_tile(uint32_t n, uint32_t row0, uint64_t seed, int shuffle, uint32_t* out_vtx_bits,
                        uint32_t* out_idx, void* stream);

/*
 * grid_quads(n) of the paper's Table 1 on the device (reference
 * pkg/src/remeshx/bench.py:42-68): 5*n*n float2 rows (4 corners + an unused
 * centre per quad) into out_vtx_bits (10*n*n words) and n*n quads
 * (5q, 5q+1, 5q+2, 5q+3) into out_idx (4*n*n words); bit-identical to the
 * reference generator.  RMX_ERANGE when 5*n*n >= 2^32.
 */
int rmx_gen_grid_quads(uint32_t n, uint32_t* out_vtx_bits, uint32_t* out_idx, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* REMESH_B200_H */
