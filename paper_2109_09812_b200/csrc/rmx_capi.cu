// rmx_capi.cu -- C-ABI entry points (include/remesh_b200.h) and the host-side
// stream orchestration of the re-indexing pipeline.  No allocation, no
// synchronisation on the hot path: every launch is stream-ordered on the
// caller's stream and reads its control words (status, plan) from device
// memory, so the whole sequence is CUDA-graph capturable.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <vector>

#include "../../include/remesh_b200.h"
#include "rmx_kernels.cuh"

namespace {

using namespace rmx;

thread_local char g_err[256] = "";

int fail_cuda(cudaError_t e, const char* what) {
    std::snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return RMX_ECUDA;
}

#define RMX_CHECK(call)                                         \
    do {                                                        \
        cudaError_t e_ = (call);                                \
        if (e_ != cudaSuccess) return fail_cuda(e_, #call);     \
    } while (0)

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

// Per-W tile sizes (rows per tile = 256 x IPT), chosen by measurement on B200.
template <int W>
struct SortIpt { static constexpr int v = W == 2 ? 16 : (W == 3 ? 16 : (W == 4 ? 20 : (W == 5 ? 16 : 2))); };
template <int W>
struct UniqIpt { static constexpr int v = W == 2 ? 16 : (W == 3 ? 12 : (W == 4 ? 8 : (W == 5 ? 8 : 2))); };

int sort_tile(int W) {
    switch (W) {
        case 2: return kBlock * SortIpt<2>::v;
        case 3: return kBlock * SortIpt<3>::v;
        case 4: return kBlock * SortIpt<4>::v;
        case 5: return kBlock * SortIpt<5>::v;
        default: return kBlock * SortIpt<0>::v;
    }
}
int uniq_tile(int W) {
    switch (W) {
        case 2: return kBlock * UniqIpt<2>::v;
        case 3: return kBlock * UniqIpt<3>::v;
        case 4: return kBlock * UniqIpt<4>::v;
        case 5: return kBlock * UniqIpt<5>::v;
        default: return kBlock * UniqIpt<0>::v;
    }
}

// warp multi-split override for tuning (RMX_RANK = match | ballot | atomic)
int rank_force() {
    static int v = [] {
        const char* e = std::getenv("RMX_RANK");
        if (!e) return -1;
        if (!std::strcmp(e, "match")) return kRankMatch;
        if (!std::strcmp(e, "ballot")) return kRankBallot;
        if (!std::strcmp(e, "atomic")) return kRankAtomic;
        return -1;
    }();
    return v;
}

// packed-key sort tiles: RMX_PK_CFG (below) selects rows per thread, tuning only
constexpr int kPkUniqIpt = 12;  // 3072-row K3' tiles (8..16 rows x 2..4 CTAs/SM measured within 1 %)
constexpr int kPkUniqTile = kBlock * kPkUniqIpt;
int pk_sort_ipt() {
    static int v = [] {
        const char* e = std::getenv("RMX_PK_CFG");
        const int x = e ? std::atoi(e) : 24;
        return (x == 12 || x == 16 || x == 20 || x == 24 || x == 28) ? x : 24;
    }();
    return v;
}
// RMX_DS=2 selects the slot-exchange downsweep (k_pk_downsweep2, rmx_packed.cuh) instead of the
// staged one: measured on C2 within -2..+10 % of the staged kernel per pass (DESIGN.md (d)), kept
// as the alternative.  RMX_DS2 = "<rows per thread>x<threads>x<CTAs per SM>" (default 16x256x3).
// Both read per call (tests switch them); the workspace is sized for the smaller tile of the two.
struct Ds2Cfg {
    int ipt, nt, minb;
};
Ds2Cfg ds2_cfg() {
    Ds2Cfg c{16, 256, 3};
    const char* e = std::getenv("RMX_DS2");
    if (e) {
        int a = 0, b = 0, m = 0;
        if (std::sscanf(e, "%dx%dx%d", &a, &b, &m) == 3) c = Ds2Cfg{a, b, m};
    }
    return c;
}
bool ds2_enabled() {
    const char* e = std::getenv("RMX_DS");
    return e && e[0] == '2';
}
int pk_sort_tile() { return ds2_enabled() ? ds2_cfg().ipt * ds2_cfg().nt : kBlock * pk_sort_ipt(); }
constexpr int kMinPkSortTile = 256 * 12;  // the smallest packed sort tile of any configuration

struct Layout {
    int D, W, P;
    uint32_t ntiles, ntiles3;
    size_t flags, rows0, rows1, map, plan;
    size_t ctl_begin, markbits, hist, vary, fields, fill, fill2, counters, desc, desc3, ctl_end;
    int bucket_shift;
    uint32_t ntiles_pk, ntiles3_pk, pk_cstride;
    size_t vals_off;  // words: origins of the packed-key path inside a row buffer
    size_t tile_counts;
    size_t pk_counts, pk_totals;  // packed passes: [256][ntiles_pk] tile counts / column scans, [256] totals
    size_t pk_digits;             // packed passes: [V] digit byte of the current pass per row
    size_t ukeys;                 // packed key of every unique row (K3' -> unpack)
    size_t rank16, vinv, vsets;   // value ranks (D <= kMaxRankDim): rank tables, inverse tables, value sets
    size_t gplan, svary, sfields; // the plan guessed from a sample of the rows, and its inputs
    size_t vsets_b;               // value sets of the odd sample blocks (saturation estimate)
    size_t vstate;                // checked value-set pass: kVstateChecked | kVstateMiss
    size_t spec;                  // speculative value-rank plan: kSpecOn | kSpecMiss (k_pack's check)
    size_t win_desc, win_counter; // window mode (rmx_window.cuh): look-back descriptors, window counter
    size_t win_rows;              // window mode: the used rows its first pass keeps
    size_t wstart, wend;          // window mode: first / one-past-last row of every window
    size_t order;                 // bit 0: the indices are not strictly increasing (k_mark)
    size_t soup;                  // soup mode: I when on (k_soup_decide), else 0
    size_t soup_prefix;           // soup mode: used rows before every packed-sort tile
    size_t rank_of;               // hash mode: new index of every candidate row
    size_t n_cand;                // hash mode: number of candidate rows
    size_t hhist, hcounters;      // hash mode: histograms and tile counters of the hashed passes
    uint32_t ntiles_hash;
    size_t repl;                  // lean: replacement row words, then a zero word (the row's index)
    bool lean;
    size_t total;
};

// lean = true: the memory-lean layout of rmx_reindex_lean (packed keys only; the caller's vertex
// buffer doubles as the second sort buffer): one 12-byte-per-row sort buffer, no AoS / hash arrays.
Layout make_layout(uint64_t V, uint32_t D, bool lean = false) {
    Layout L{};
    L.lean = lean;
    L.D = static_cast<int>(D);
    L.W = L.D + 1;
    L.P = 4 * L.D;
    L.ntiles = static_cast<uint32_t>((V + sort_tile(L.W) - 1) / sort_tile(L.W));
    L.ntiles3 = static_cast<uint32_t>((V + uniq_tile(L.W) - 1) / uniq_tile(L.W));
    L.ntiles_pk = static_cast<uint32_t>((V + pk_sort_tile() - 1) / pk_sort_tile());
    L.ntiles3_pk = static_cast<uint32_t>((V + kPkUniqTile - 1) / kPkUniqTile);
    L.vals_off = (static_cast<size_t>(V) * (L.D >= 2 ? 2 : 1) + 3) & ~static_cast<size_t>(3);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t at = off;
        off = align_up(off + bytes);
        return at;
    };
    const size_t row_bytes = static_cast<size_t>(V) * (lean ? 3 : L.W) * 4 + 256;  // slack: bulk copies round up
    L.flags = take(V);
    L.rows0 = take(row_bytes);
    L.rows1 = take(lean ? 0 : row_bytes);
    L.map = take(static_cast<size_t>(V) * 4);
    L.plan = take(plan_words(L.P) * 4);
    L.pk_cstride = (L.ntiles_pk + kUpGroup - 1) / kUpGroup * kUpGroup;
    const size_t max_tiles_pk = (V + kMinPkSortTile - 1) / kMinPkSortTile + kUpGroup;  // any tile choice
    L.pk_counts = take(max_tiles_pk * 256 * 4);
    L.pk_totals = take(256 * 4);
    L.pk_digits = take(2 * (align_up(static_cast<size_t>(V) + 16)));  // two arrays: this pass's, the next's
    L.ukeys = take(static_cast<size_t>(V) * 8);  // packed: unique keys; hash: (group, origin) per row
    L.ntiles_hash = static_cast<uint32_t>((V + kHashTile - 1) / kHashTile);
    const bool hash = !lean && L.D >= 3 && L.D <= kHashMaxDim;
    L.rank_of = take(hash ? static_cast<size_t>(V) * 4 : 0);
    const size_t vr_dim = L.D <= kMaxRankDim ? static_cast<size_t>(L.D) : 0;
    L.rank16 = take(vr_dim * (size_t{1} << kMaxValueBits) * 2);
    L.vinv = take(vr_dim * (size_t{1} << kMaxValueBits) * 2);
    L.gplan = take(plan_words(L.P) * 4);
    L.ctl_begin = off;
    L.vsets = take(vr_dim * kValueWords * 4);
    L.vsets_b = take(vr_dim * kValueWords * 4);
    L.svary = take(vr_dim * 4);
    L.vstate = take(16);
    L.n_cand = take(16);
    L.hhist = take(kHashPasses * 256 * 4);
    L.hcounters = take(kHashPasses * 4 + 16);
    L.spec = take(16);
    L.win_desc = take(static_cast<size_t>(kWinCount) * 8);  // window mode: look-back descriptors
    L.win_counter = take(16);
    L.win_rows = take(16);
    L.order = take(16);
    L.soup = take(16);
    L.sfields = take(vr_dim * kFieldWords * 4);
    L.markbits = take((static_cast<size_t>(V) + 31) / 32 * 4 + 16);
    L.hist = take(static_cast<size_t>(L.P) * 256 * 4);
    L.vary = take(static_cast<size_t>(L.D) * 4);
    L.fields = take(static_cast<size_t>(L.D) * kFieldWords * 4);
    L.fill = take(256 * 4);
    L.fill2 = take(256 * 4);
    int bits = 0;
    while (bits < 40 && (1ull << bits) < V) ++bits;
    L.bucket_shift = bits > 8 ? bits - 8 : 0;
    L.counters = take(static_cast<size_t>(L.P + 2 + kMaxPackedPasses + 1) * 4);
    L.desc = take(lean ? 256 : static_cast<size_t>(L.ntiles > max_tiles_pk ? L.ntiles : max_tiles_pk) * 256 * 8);
    L.desc3 = take(lean ? 256 : static_cast<size_t>(L.ntiles3) * 8);
    L.repl = take((RMX_MAX_DIM + 4) * 4);  // lean: the replacement row (the vertex buffer is overwritten)
    L.tile_counts = take(static_cast<size_t>(L.ntiles3_pk) * 4);
    L.wstart = take(static_cast<size_t>(kWinCount) * 4);
    L.wend = take(static_cast<size_t>(kWinCount) * 4);
    L.soup_prefix = take(static_cast<size_t>(max_tiles_pk) * 4);
    L.ctl_end = off;
    L.total = off;
    return L;
}

// ---- per-device cached launch facts -------------------------------------
struct DeviceFacts {
    int sms = 0;
};
std::mutex g_mu;
DeviceFacts g_dev[64];

int device_sms(int& sms) {
    int dev = 0;
    RMX_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_mu);
    if (dev < 0 || dev >= 64) return fail_cuda(cudaErrorInvalidDevice, "device id");
    if (g_dev[dev].sms == 0) RMX_CHECK(cudaDeviceGetAttribute(&g_dev[dev].sms, cudaDevAttrMultiProcessorCount, dev));
    sms = g_dev[dev].sms;
    return RMX_OK;
}

// Opt a kernel in to `smem` bytes of dynamic shared memory on the current
// device.  The attribute only ever grows: calls on other threads with a
// smaller need (another dim, a smaller mesh) must not shrink it under a
// launch that is about to use more.
std::mutex g_attr_mu;
struct SmemAttr {
    const void* fn;
    int dev;
    size_t bytes;
};
std::vector<SmemAttr> g_attr;

template <typename K>
int ensure_smem(K kernel, size_t smem) {
    if (smem <= 32 * 1024) return RMX_OK;  // (dynamic + static above 48 KB needs the opt-in)
    int dev = 0;
    RMX_CHECK(cudaGetDevice(&dev));
    const void* fn = reinterpret_cast<const void*>(kernel);
    std::lock_guard<std::mutex> lk(g_attr_mu);
    for (SmemAttr& e : g_attr) {
        if (e.fn == fn && e.dev == dev) {
            if (e.bytes < smem) {
                RMX_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
                e.bytes = smem;
            }
            return RMX_OK;
        }
    }
    RMX_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    g_attr.push_back(SmemAttr{fn, dev, smem});
    return RMX_OK;
}

// Persistent grid size for a kernel: resident CTAs per SM x SMs.
template <typename K>
int persistent_grid(K kernel, size_t smem, uint64_t work_items, int& grid, int threads = kBlock) {
    int sms = 0;
    int rc = device_sms(sms);
    if (rc) return rc;
    if ((rc = ensure_smem(kernel, smem))) return rc;
    int per_sm = 0;
    RMX_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
    if (per_sm < 1) per_sm = 1;
    uint64_t g = static_cast<uint64_t>(per_sm) * sms;
    if (work_items < g) g = work_items;
    grid = static_cast<int>(g < 1 ? 1 : g);
    return RMX_OK;
}

int grid_for_stream(uint64_t items, int& grid);

// ---- launches ------------------------------------------------------------------
// run_pipeline launches its kernels with programmatic stream serialization
// (each kernel starts with pdl_enter(), rmx_common.cuh): the next kernel's
// launch and CTA ramp-up overlap the previous kernel's tail.  Off while a
// graph is captured and with RMX_PDL=0.
thread_local bool t_pdl = false;

bool pdl_enabled() {
    const char* e = std::getenv("RMX_PDL");  // read per call: tests switch it at run time
    return !(e && e[0] == '0');
}

struct PdlScope {
    explicit PdlScope(bool on) { t_pdl = on; }
    ~PdlScope() { t_pdl = false; }
};

// kernels launched by this process through the pipeline (rmx_kernel_launches_total)
std::atomic<unsigned long long> g_launches{0};

template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = t_pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// ---- kernel dispatch by compile-time width --------------------------------
template <int D_CT>
int launch_build(const BuildArgs& a, cudaStream_t s) {
    const size_t smem = 0;
    int grid = 0;
    int rc = persistent_grid(k_build_rows<D_CT>, smem, (static_cast<uint64_t>(a.n) + kBlock - 1) / kBlock, grid);
    if (rc) return rc;
    RMX_CHECK(launch(k_build_rows<D_CT>, grid, kBlock, smem, s, a));
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

template <int W_CT, int IPT>
int launch_pass(const SortArgs& a, cudaStream_t s) {
    auto kern = k_sort_pass<W_CT, IPT>;
    const size_t smem = SortTraits<W_CT, IPT>::smem_bytes(a.dim + 1);
    int grid = 0;
    int rc = persistent_grid(kern, smem, a.ntiles, grid);
    if (rc) return rc;
    RMX_CHECK(launch(kern, grid, kBlock, smem, s, a));
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

template <int W_CT, int IPT>
int launch_unique(const UniqueArgs& a, cudaStream_t s) {
    auto kern = k_unique<W_CT, IPT>;
    const size_t smem = UniqueTraits<W_CT, IPT>::smem_bytes(a.dim + 1);
    int grid = 0;
    int rc = persistent_grid(kern, smem, a.ntiles, grid);
    if (rc) return rc;
    RMX_CHECK(launch(kern, grid, kBlock, smem, s, a));
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

template <int D_CT>
int launch_vary(const VaryArgs& a, cudaStream_t s) {
    int grid = 0;
    int rc = persistent_grid(k_vary<D_CT>, 0, (static_cast<uint64_t>(a.n) + kBlock - 1) / kBlock, grid);
    if (rc) return rc;
    RMX_CHECK(launch(k_vary<D_CT>, grid, kBlock, 0, s, a));
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

int dispatch_vary(const VaryArgs& a, cudaStream_t s) {
    switch (a.dim) {
        case 1: return launch_vary<1>(a, s);
        case 2: return launch_vary<2>(a, s);
        case 3: return launch_vary<3>(a, s);
        case 4: return launch_vary<4>(a, s);
        default: return launch_vary<0>(a, s);
    }
}

template <int D_CT>
int launch_pack(const PackArgs& a, cudaStream_t s, bool with_check) {
    int grid = 0;
    int rc = persistent_grid(k_pack<D_CT>, 0, (static_cast<uint64_t>(a.n) + kBlock - 1) / kBlock, grid);
    if (rc) return rc;
    RMX_CHECK(launch(k_pack<D_CT>, grid, kBlock, 0, s, a));
    RMX_CHECK(cudaGetLastError());
    if constexpr (D_CT >= 1 && D_CT <= kMaxRankDim) {
        if (with_check) {  // speculative plans: the checking variant (the plain one exited then)
            RMX_CHECK(launch(k_pack<D_CT, true>, grid, kBlock, 0, s, a));
            RMX_CHECK(cudaGetLastError());
        }
    }
    return RMX_OK;
}

// RMX_VALUE_RANK=0 turns value ranks off (read per call: tests switch it at run time)
bool value_rank_enabled() {
    const char* e = std::getenv("RMX_VALUE_RANK");
    return !(e && e[0] == '0');
}

// Value ranks cost the sample kernels and one read of the vertices; a saved 8-bit pass pays for
// that from ~2^25 rows on (C1, 3.15M rows: 0.37 ms with, 0.36 without; grid_quads(1024), 5.2M
// rows ranked to 3 passes: 0.44 vs 0.36 ms).  RMX_VALUE_RANK_MIN overrides the row count (tests).
uint64_t value_rank_min_rows() {
    const char* e = std::getenv("RMX_VALUE_RANK_MIN");
    return e ? std::strtoull(e, nullptr, 10) : (1ull << 25);
}

template <int D_CT>
int launch_valueset(const ValueSetArgs& a, uint64_t items, cudaStream_t s) {
    int sms = 0;
    int rc = device_sms(sms);
    if (rc) return rc;
    const size_t smem = kValueSetBytes + 16;  // + a spare byte for the components that are not candidates
    if ((rc = ensure_smem(k_valueset<D_CT>, smem))) return rc;
    const uint64_t want = (items + kVsThreads - 1) / kVsThreads;
    const int grid = static_cast<int>(want < static_cast<uint64_t>(sms) ? (want ? want : 1) : sms);
    RMX_CHECK(launch(k_valueset<D_CT>, grid, kVsThreads, smem, s, a));
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

int dispatch_valueset(const ValueSetArgs& a, int dim, cudaStream_t s) {
    const uint64_t items = a.shift ? (static_cast<uint64_t>(a.n) >> a.shift) + 256 : a.n;
    switch (dim) {
        case 1: return launch_valueset<1>(a, items, s);
        case 2: return launch_valueset<2>(a, items, s);
        case 3: return launch_valueset<3>(a, items, s);
        case 4: return launch_valueset<4>(a, items, s);
        default: return RMX_OK;
    }
}

int dispatch_pack(const PackArgs& a, cudaStream_t s, bool with_check = false) {
    switch (a.dim) {
        case 1: return launch_pack<1>(a, s, with_check);
        case 2: return launch_pack<2>(a, s, with_check);
        case 3: return launch_pack<3>(a, s, with_check);
        case 4: return launch_pack<4>(a, s, with_check);
        default: return launch_pack<0>(a, s, false);
    }
}

constexpr int kCommonPasses = 5;

template <int IPT, int MINB>
int launch_downsweep(const SortPkArgs& a, cudaStream_t s) {
    const size_t smem = SortPkTraits<IPT>::smem_bytes();
    int rc = ensure_smem(k_pk_downsweep<IPT, MINB>, smem);
    if (rc) return rc;
    // passes past kCommonPasses run only for > 40-bit keys: 4 tiles per CTA there, so that when
    // they do not run (the common case) the exiting grid is a quarter the size
    // (window mode's fallback passes: 16 tiles per CTA -- they rarely run)
    const uint32_t tpc = a.win_fb ? 16u : a.pass >= kCommonPasses ? 4u : 1u;
    RMX_CHECK(launch(k_pk_downsweep<IPT, MINB>, (a.ntiles + tpc - 1) / tpc, kBlock, smem, s, a, tpc));
    RMX_CHECK(cudaGetLastError());
    if (a.pass == 2 && !a.win_fb) {  // window mode's first pass when it drops the unused rows (no soup
                                     // mode): its own instantiation, 16 tiles per CTA (a small exiting grid)
        if ((rc = ensure_smem(k_pk_downsweep<IPT, MINB, true>, smem))) return rc;
        RMX_CHECK(launch(k_pk_downsweep<IPT, MINB, true>, (a.ntiles + 15) / 16, kBlock, smem, s, a, 16u));
        RMX_CHECK(cudaGetLastError());
    }
    return RMX_OK;
}

// RMX_PK_CFG = "<rows per thread>x<CTAs per SM>" (tuning aid; default 24x2: 6144-row tiles,
// two CTAs per SM -- measured against 8..32 rows x 1..4 CTAs on C2 / C3 / C5s)
int pk_minb() {
    static int v = [] {
        const char* e = std::getenv("RMX_PK_CFG");
        const char* x = e ? std::strchr(e, 'x') : nullptr;
        return x ? std::atoi(x + 1) : 2;
    }();
    return v;
}

template <int IPT, int NT, int MINB>
int launch_downsweep2(const SortPkArgs& a, cudaStream_t s) {
    constexpr size_t smem = SortPk2Traits<2, IPT, NT>::smem_bytes();  // sized for u64 keys
    int rc = ensure_smem(k_pk_downsweep2<IPT, NT, MINB>, smem);
    if (rc) return rc;
    RMX_CHECK(launch(k_pk_downsweep2<IPT, NT, MINB>, a.ntiles, NT, smem, s, a));
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

int launch_sort_pk(const SortPkArgs& a, cudaStream_t s) {
    int grid = 0;
    int rc = grid_for_stream(static_cast<uint64_t>((a.ntiles + kUpGroup - 1) / kUpGroup) * kBlock, grid);
    if (rc) return rc;
    RMX_CHECK(launch(k_pk_upsweep<false>, grid, kBlock, 0, s, a, static_cast<uint32_t>(pk_sort_tile())));
    RMX_CHECK(cudaGetLastError());
    if (a.pass == 2 && !a.win_fb) {  // window mode's dropping first pass (see launch_downsweep)
        RMX_CHECK(launch(k_pk_upsweep<true>, grid, kBlock, 0, s, a, static_cast<uint32_t>(pk_sort_tile())));
        RMX_CHECK(cudaGetLastError());
    }
    RMX_CHECK(launch(k_pk_colscan, 256, 1024, 0, s, a));
    RMX_CHECK(cudaGetLastError());
    if (ds2_enabled()) {
        const Ds2Cfg c = ds2_cfg();
        switch (c.ipt * 10000 + c.nt * 10 + c.minb) {
            case 240000 + 2562: return launch_downsweep2<24, 256, 2>(a, s);
            case 160000 + 2563: return launch_downsweep2<16, 256, 3>(a, s);
            case 120000 + 2564: return launch_downsweep2<12, 256, 4>(a, s);
            case 80000 + 5123: return launch_downsweep2<8, 512, 3>(a, s);
            case 160000 + 5122: return launch_downsweep2<16, 512, 2>(a, s);
            default: return launch_downsweep2<12, 512, 2>(a, s);
        }
    }
    const int cfg = pk_sort_ipt() * 10 + pk_minb();
    switch (cfg) {
        case 123: return launch_downsweep<12, 3>(a, s);
        case 162: return launch_downsweep<16, 2>(a, s);
        case 202: return launch_downsweep<20, 2>(a, s);
        case 282: return launch_downsweep<28, 2>(a, s);
        default: return launch_downsweep<24, 2>(a, s);
    }
}

int launch_unique_pk(const UniquePkArgs& a, cudaStream_t s) {
    const size_t smem = UniquePkTraits<kPkUniqIpt>::smem_bytes();
    int grid = 0;
    int rc = persistent_grid(k_unique_pk<kPkUniqIpt>, smem, a.ntiles, grid);
    if (rc) return rc;
    RMX_CHECK(launch(k_unique_pk<kPkUniqIpt>, grid, kBlock, smem, s, a));
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

template <int D_CT>
int launch_unpack_pk_d(const UnpackPkArgs& a, uint64_t max_rows, cudaStream_t s) {
    int grid = 0;
    int rc = grid_for_stream(max_rows, grid);
    if (rc) return rc;
    RMX_CHECK(launch(k_unpack_pk<D_CT>, grid, kBlock, 0, s, a));
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

int launch_unpack_pk(const UnpackPkArgs& a, uint64_t max_rows, cudaStream_t s) {
    switch (a.dim) {
        case 1: return launch_unpack_pk_d<1>(a, max_rows, s);
        case 2: return launch_unpack_pk_d<2>(a, max_rows, s);
        case 3: return launch_unpack_pk_d<3>(a, max_rows, s);
        case 4: return launch_unpack_pk_d<4>(a, max_rows, s);
        default: return launch_unpack_pk_d<0>(a, max_rows, s);
    }
}

int dispatch_build(const BuildArgs& a, cudaStream_t s) {
    switch (a.dim) {
        case 1: return launch_build<1>(a, s);
        case 2: return launch_build<2>(a, s);
        case 3: return launch_build<3>(a, s);
        case 4: return launch_build<4>(a, s);
        default: return launch_build<0>(a, s);
    }
}

int dispatch_pass(const SortArgs& a, cudaStream_t s) {
    switch (a.dim + 1) {
        case 2: return launch_pass<2, SortIpt<2>::v>(a, s);
        case 3: return launch_pass<3, SortIpt<3>::v>(a, s);
        case 4: return launch_pass<4, SortIpt<4>::v>(a, s);
        case 5: return launch_pass<5, SortIpt<5>::v>(a, s);
        default: return launch_pass<0, SortIpt<0>::v>(a, s);
    }
}

int dispatch_unique(const UniqueArgs& a, cudaStream_t s) {
    switch (a.dim + 1) {
        case 2: return launch_unique<2, UniqIpt<2>::v>(a, s);
        case 3: return launch_unique<3, UniqIpt<3>::v>(a, s);
        case 4: return launch_unique<4, UniqIpt<4>::v>(a, s);
        case 5: return launch_unique<5, UniqIpt<5>::v>(a, s);
        default: return launch_unique<0, UniqIpt<0>::v>(a, s);
    }
}

int grid_for_stream(uint64_t items, int& grid) {
    int sms = 0;
    int rc = device_sms(sms);
    if (rc) return rc;
    uint64_t g = (items + kBlock - 1) / kBlock;
    const uint64_t cap = static_cast<uint64_t>(sms) * 16;
    if (g > cap) g = cap;
    grid = static_cast<int>(g < 1 ? 1 : g);
    return RMX_OK;
}

struct Recorder {
    void* const* events;
    int n;
    int k = 0;
    cudaStream_t s;
    int mark() {
        if (events && k < n && events[k]) RMX_CHECK(cudaEventRecord(static_cast<cudaEvent_t>(events[k]), s));
        ++k;
        return RMX_OK;
    }
};

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// the AoS rows path can only be chosen when more than 64 key bits may vary
bool aos_possible(int D) { return 32 * D > 64; }
// packed passes that can run: ceil(32 D / 8) digits, at most kMaxPackedPasses
int packed_passes_max(int D) { return 4 * D < kMaxPackedPasses ? 4 * D : kMaxPackedPasses; }

// small meshes take the one-CTA path (RMX_SMALL=0 forces the large-mesh pipeline, for tests)
bool small_path(uint64_t V, uint32_t D, uint64_t I) {
    if (V < 1 || V > kSmallV || D > kSmallD || V * D > kSmallWords || I > kSmallI) return false;
    const char* e = std::getenv("RMX_SMALL");  // read per call: tests switch it at run time
    return !(e && e[0] == '0');
}

// ---- graph launch path ------------------------------------------------------
// rmx_graph_create captures run_pipeline on a capturing stream (plain capture: every kernel
// checks the device plan and exits when its section does not apply; the programmatic launch
// dependencies become graph edges).
constexpr cudaStreamCaptureMode kCaptureMode = cudaStreamCaptureModeThreadLocal;

// hash mode (rmx_hash.cuh) for keys wider than 64 bits: D in [3, kHashMaxDim]; RMX_HASH=0 turns it
// off (read per call: tests switch it at run time)
bool hash_possible(int D) { return D >= 3 && D <= kHashMaxDim; }
// RMX_WINDOW=0: no window mode (rmx_window.cuh; A/B)
bool win_enabled() {
    const char* e = std::getenv("RMX_WINDOW");
    return !(e && e[0] == '0');
}
// RMX_SOUP=0: no soup mode (strictly increasing indices: map fill into the output indices, no
// remap; A/B)
bool soup_enabled() {
    const char* e = std::getenv("RMX_SOUP");
    return !(e && e[0] == '0');
}
// RMX_SPEC=0: no speculative value-rank plans.  Speculation is used for D <= 3: the checking k_pack
// costs less than the full value-set pass there (C2 7.34 -> 6.95 ms), not for D = 4 (C3 4.71 -> 4.82) (always the full value-set pass; A/B)
bool spec_enabled() {
    const char* e = std::getenv("RMX_SPEC");
    return !(e && e[0] == '0');
}
// RMX_HASH_RAW=0: build the hash-mode rows in a separate pass (A/B)
bool hash_raw_enabled() {
    const char* e = std::getenv("RMX_HASH_RAW");
    return !(e && e[0] == '0');
}
bool hash_enabled() {
    const char* e = std::getenv("RMX_HASH");
    return !(e && e[0] == '0');
}

template <int D_CT>
int launch_hash_build_d(const HashArgs& a, cudaStream_t s) {
    int grid = 0;
    int rc = persistent_grid(k_hash_build<D_CT>, 0, (static_cast<uint64_t>(a.n) + kBlock - 1) / kBlock, grid);
    if (rc) return rc;
    RMX_CHECK(launch(k_hash_build<D_CT>, grid, kBlock, 0, s, a));
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

int dispatch_hash_build(const HashArgs& a, cudaStream_t s) {
    switch (a.dim) {
        case 3: return launch_hash_build_d<3>(a, s);
        case 4: return launch_hash_build_d<4>(a, s);
        default: return launch_hash_build_d<0>(a, s);
    }
}

template <int W_CT, int IPT, bool RAW = false, bool SOUP = false>
int launch_hashed_pass(const SortArgs& a, cudaStream_t s) {
    auto kern = k_sort_pass<W_CT, IPT, true, RAW, SOUP>;
    const size_t smem = SortTraits<W_CT, IPT>::smem_bytes(a.dim + 1);
    int grid = 0;
    int rc = persistent_grid(kern, smem, a.ntiles, grid);
    if (rc) return rc;
    RMX_CHECK(launch(kern, grid, kBlock, smem, s, a));
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

template <int D_CT>
int launch_hash_dedup_d(const HashArgs& a, cudaStream_t s) {
    const size_t smem = hash_dedup_smem(a.dim);
    int rc = ensure_smem(k_hash_dedup<D_CT>, smem);
    if (rc) return rc;
    int grid = 0;
    if ((rc = persistent_grid(k_hash_dedup<D_CT>, smem, a.ntiles, grid))) return rc;
    RMX_CHECK(launch(k_hash_dedup<D_CT>, grid, kBlock, smem, s, a));
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

// the two hashed passes (rows0 -> rows1 -> rows0) and the per-tile dedup
int launch_hash_groups(const HashArgs& ha, SortArgs sa, cudaStream_t s) {
    int rc = RMX_OK;
    for (int hp = 0; hp < kHashPasses && rc == RMX_OK; ++hp) {
        sa.pass = hp;
        switch (ha.dim) {
            case 3:
                if (hp == 0 && ha.hist_only) {  // the raw pass: plain and soup-mode variants (one runs)
                    rc = launch_hashed_pass<4, SortIpt<4>::v, true>(sa, s);
                    if (!rc) rc = launch_hashed_pass<4, SortIpt<4>::v, true, true>(sa, s);
                } else {
                    rc = launch_hashed_pass<4, SortIpt<4>::v>(sa, s);
                }
                break;
            case 4: rc = launch_hashed_pass<5, SortIpt<5>::v>(sa, s); break;
            default: rc = launch_hashed_pass<0, SortIpt<0>::v>(sa, s); break;
        }
    }
    if (rc) return rc;
    switch (ha.dim) {
        case 3: return launch_hash_dedup_d<3>(ha, s);
        case 4: return launch_hash_dedup_d<4>(ha, s);
        default: return launch_hash_dedup_d<0>(ha, s);
    }
}

// lean (rmx_reindex_lean): `vtx` is overwritten (it becomes the second sort buffer after k_pack has
// read it), out_vtx is ignored -- the unique rows land in the final sort buffer, *d_where = 0
// (workspace rows0) or 1 (the vertex buffer) --, only packed keys are supported (a plan that is not
// packed sets RMX_STATUS_LEAN_UNSUPPORTED and the remaining kernels exit).
int run_pipeline(const uint32_t* vtx, uint64_t V, uint32_t D, const uint32_t* idx, uint64_t E, uint32_t K,
                 uint32_t* out_vtx, uint32_t* out_idx, uint64_t* d_count, uint32_t* d_status, void* ws,
                 size_t ws_bytes, const rmx_scratch* sc, cudaStream_t s, void* const* events, int n_events,
                 bool lean = false, uint32_t* d_where = nullptr) {
    g_err[0] = '\0';
    if (lean && (D < 3 || (V & 1u) || sc || !d_where || V <= kSmallV)) {
        std::snprintf(g_err, sizeof(g_err), "lean mode needs dim >= 3, an even vertex count > %u, no scratch",
                      static_cast<unsigned>(kSmallV));
        return RMX_EINVAL;
    }
    if (D < 1 || K < 1) {
        std::snprintf(g_err, sizeof(g_err), "dim and arity must be >= 1 (got %u, %u)", D, K);
        return RMX_EINVAL;
    }
    if (D > RMX_MAX_DIM) {
        std::snprintf(g_err, sizeof(g_err), "dim %u exceeds the CUDA path limit %d", D, RMX_MAX_DIM);
        return RMX_EINVAL;
    }
    if (V >= (1ull << 32)) {
        std::snprintf(g_err, sizeof(g_err), "vertex count %llu exceeds 32-bit index range",
                      static_cast<unsigned long long>(V));
        return RMX_ERANGE;
    }
    if (!d_count || !d_status) {
        std::snprintf(g_err, sizeof(g_err), "d_new_count and d_status are required");
        return RMX_EINVAL;
    }
    const uint64_t I = E * K;
    Recorder rec{events, n_events, 0, s};
    int rc = rec.mark();
    if (rc) return rc;
    RMX_CHECK(cudaMemsetAsync(d_count, 0, sizeof(uint64_t), s));
    RMX_CHECK(cudaMemsetAsync(d_status, 0, sizeof(uint32_t), s));
    if (E == 0) {  // pipeline.py:142-146: every vertex unused, empty result
        if (sc && sc->is_used && V) RMX_CHECK(cudaMemsetAsync(sc->is_used, 0, V, s));
        return RMX_OK;
    }
    if ((V && !vtx) || !idx || !out_idx || (V && !out_vtx && !lean)) {
        std::snprintf(g_err, sizeof(g_err), "null buffer");
        return RMX_EINVAL;
    }
    if (reinterpret_cast<uintptr_t>(ws) % kAlign) {  // bulk copies and 16-byte loads of workspace arrays
        std::snprintf(g_err, sizeof(g_err), "workspace must be %zu-byte aligned", kAlign);
        return RMX_EINVAL;
    }
    const PdlScope pdl(pdl_enabled());
    const Layout L = make_layout(V, D, lean);
    if (!ws || ws_bytes < L.total) {
        std::snprintf(g_err, sizeof(g_err), "workspace %zu bytes < required %zu", ws_bytes, L.total);
        return RMX_ENOSPC;
    }
    if (small_path(V, D, I)) {  // one CTA does it all (rmx_small.cuh)
        const size_t smem = small_smem_bytes(static_cast<uint32_t>(V), D);
        if ((rc = ensure_smem(k_small, smem))) return rc;
        SmallArgs a{vtx, static_cast<uint32_t>(V), D, idx, I, out_vtx, out_idx,
                    reinterpret_cast<unsigned long long*>(d_count), d_status, sc ? *sc : rmx_scratch{}};
        g_launches.fetch_add(1, std::memory_order_relaxed);
        k_small<<<1, kSmallThreads, smem, s>>>(a);
        RMX_CHECK(cudaGetLastError());
        while (rec.k < rec.n) {  // stage events of a profiled call: all at the end
            if ((rc = rec.mark())) return rc;
        }
        return RMX_OK;
    }
    char* base = static_cast<char*>(ws);
    uint8_t* flags = (sc && sc->is_used) ? sc->is_used : reinterpret_cast<uint8_t*>(base + L.flags);
    uint32_t* rows0 = reinterpret_cast<uint32_t*>(base + L.rows0);
    // lean: the vertex buffer is the second sort buffer once k_pack has read it
    uint32_t* rows1 = lean ? const_cast<uint32_t*>(vtx) : reinterpret_cast<uint32_t*>(base + L.rows1);
    uint32_t* map = reinterpret_cast<uint32_t*>(base + L.map);
    uint32_t* plan = reinterpret_cast<uint32_t*>(base + L.plan);
    uint32_t* hist = reinterpret_cast<uint32_t*>(base + L.hist);
    uint32_t* vary = reinterpret_cast<uint32_t*>(base + L.vary);
    uint32_t* fields = reinterpret_cast<uint32_t*>(base + L.fields);
    uint32_t* counters = reinterpret_cast<uint32_t*>(base + L.counters);
    uint64_t* desc = reinterpret_cast<uint64_t*>(base + L.desc);
    uint64_t* desc3 = reinterpret_cast<uint64_t*>(base + L.desc3);

    RMX_CHECK(cudaMemsetAsync(base + L.ctl_begin, 0, L.ctl_end - L.ctl_begin, s));
    RMX_CHECK(cudaMemsetAsync(base + L.wstart, 0xFF, static_cast<size_t>(kWinCount) * 4, s));
    if (V) RMX_CHECK(cudaMemsetAsync(flags, 0, V, s));

    // K1 mark (byte flags for in-order indices, a bit set for scattered ones), then merge them
    {
        uint32_t* bits = reinterpret_cast<uint32_t*>(base + L.markbits);
        MarkArgs a{idx, I, V, flags, bits, d_status, aligned16(idx) ? 1 : 0,
                   reinterpret_cast<uint32_t*>(base + L.order)};
        int grid = 0;
        rc = grid_for_stream(a.vec ? (I + 3) / 4 : I, grid);
        if (rc) return rc;
        RMX_CHECK(launch(k_mark, grid, kBlock, 0, s, a));
        RMX_CHECK(cudaGetLastError());
        if (V) {
            rc = grid_for_stream((V + 31) / 32, grid);
            if (rc) return rc;
            RMX_CHECK(launch(k_expand_marks, grid, kBlock, 0, s, bits, V, flags));
            RMX_CHECK(cudaGetLastError());
        }
    }
    if ((rc = rec.mark())) return rc;
    if (V == 0) {  // every index is out of range; status is set
        return RMX_OK;
    }
    // hash mode (rmx_hash.cuh) replaces the whole-set AoS sort unless the caller wants the scratch
    // arrays of the stable sort (org_id, perm: only the AoS path produces them) or RMX_HASH=0
    const bool hash_ok = !lean && hash_possible(L.D) && sc == nullptr && hash_enabled();
    // K1a varying bits of the cleaned vertex set, then the plan (packed, hash or AoS)
    const int vec = (aligned16(vtx) && aligned16(flags)) ? 1 : 0;
    const bool value_ranks = L.D <= kMaxRankDim && value_rank_enabled() && V >= value_rank_min_rows();
    uint32_t* gplan = reinterpret_cast<uint32_t*>(base + L.gplan);
    uint32_t* svary = reinterpret_cast<uint32_t*>(base + L.svary);
    uint32_t* sfields = reinterpret_cast<uint32_t*>(base + L.sfields);
    uint32_t* vsets = reinterpret_cast<uint32_t*>(base + L.vsets);
    if (value_ranks) {
        // value ranks: K1a over a sample -> guessed plan -> the sample's value sets -> worth it?
        // -> one full pass: exact K1a outputs + (if worth it) every used row's values
        // (the full pass checks the rows against the sample instead of recomputing K1a when it
        // collects values; k_vary then copies the sample's outputs, or computes them when the
        // pass found a row outside the sample or did not run)
        const uint32_t shift = V >= (1ull << 22) ? 6u : 0u;
        uint32_t* vstate = reinterpret_cast<uint32_t*>(base + L.vstate);
        uint32_t* spec = reinterpret_cast<uint32_t*>(base + L.spec);
        VaryArgs sa{vtx, flags, idx, svary, sfields, d_status, static_cast<uint32_t>(V), L.D, vec, shift,
                    nullptr, nullptr, nullptr, nullptr};
        if ((rc = dispatch_vary(sa, s))) return rc;
        RMX_CHECK(launch(k_plan, 1, 32, 0, s, svary, sfields, gplan, L.D, d_status, 0, nullptr));
        uint32_t* vsets_b = reinterpret_cast<uint32_t*>(base + L.vsets_b);
        ValueSetArgs va{vtx, flags, idx, gplan, sfields, vsets, svary, vstate, d_status, static_cast<uint32_t>(V),
                        shift, vec, 0, gplan, 0, spec, 0};
        if (shift) {  // the sample's value sets, even blocks into vsets and odd blocks into vsets_b
            if ((rc = dispatch_valueset(va, L.D, s))) return rc;
            ValueSetArgs vb_args = va;
            vb_args.vsets = vsets_b;
            vb_args.parity = 1;
            if ((rc = dispatch_valueset(vb_args, L.D, s))) return rc;
        }
        // (with two sample halves that saw the same value sets: speculate, kSpecOn)
        ValuePlanArgs pd{gplan, vsets, shift ? vsets_b : nullptr, nullptr, nullptr, d_status, L.D, 0, nullptr,
                         nullptr, svary, nullptr, nullptr, nullptr, spec, vstate, spec_enabled() && L.D <= 3 ? 1 : 0,
                         0};
        RMX_CHECK(launch(k_value_plan, 1, 1024, 0, s, pd));
        va.shift = 0u;
        if ((rc = dispatch_valueset(va, L.D, s))) return rc;
        // decide again on the full pass's value sets (tight lower bounds even where a row fell
        // outside the sample): the second chance below runs only if value ranks can still pay
        pd.vsets_b = nullptr;
        RMX_CHECK(launch(k_value_plan, 1, 1024, 0, s, pd));
        VaryArgs fa{vtx, flags, idx, vary, fields, d_status, static_cast<uint32_t>(V), L.D, vec, 0u,
                    vstate, svary, sfields, nullptr};
        if ((rc = dispatch_vary(fa, s))) return rc;
    } else {
        VaryArgs a{vtx, flags, idx, vary, fields, d_status, static_cast<uint32_t>(V), L.D, vec, 0u,
                   nullptr, nullptr, nullptr, nullptr};
        if ((rc = dispatch_vary(a, s))) return rc;
    }
    if ((rc = rec.mark())) return rc;
    RMX_CHECK(launch(k_plan, 1, 32, 0, s, vary, fields, plan, L.D, d_status, hash_ok ? 1 : 0, nullptr));
    RMX_CHECK(cudaGetLastError());
    // soup mode (rmx_packed.cuh k_soup_decide): strictly increasing indices + a packed plan; not with
    // scratch (org_id holds origins), lean mode or the slot-exchange downsweep
    uint32_t* soup = reinterpret_cast<uint32_t*>(base + L.soup);
    uint32_t* win_rows = reinterpret_cast<uint32_t*>(base + L.win_rows);  // window mode (rmx_window.cuh)
    uint32_t* soup_prefix = reinterpret_cast<uint32_t*>(base + L.soup_prefix);
    const uint32_t* order = reinterpret_cast<const uint32_t*>(base + L.order);
    const int soup_ok = (!lean && sc == nullptr && soup_enabled() && !ds2_enabled()) ? 1 : 0;
    // hash mode, float3 with aligned vertices: the first hashed pass stages the vertices itself and
    // k_hash_build only counts the hashed digits (no row build: 16 B per row less written and read)
    const int hash_raw = (L.D == 3 && vec && hash_raw_enabled()) ? 1 : 0;
    auto launch_soup = [&](const uint32_t* gate) -> int {
        RMX_CHECK(launch(k_soup_decide, 1, 32, 0, s, static_cast<const uint32_t*>(plan), order, soup,
                         static_cast<uint32_t>(I), L.D, soup_ok, hash_raw, static_cast<const uint32_t*>(d_status),
                         gate));
        int g = 0;
        int rc2 = grid_for_stream(L.ntiles_pk, g);
        if (rc2) return rc2;
        RMX_CHECK(launch(k_soup_prefix, g, kBlock, 0, s, idx, static_cast<uint32_t>(I),
                         static_cast<const uint32_t*>(soup), soup_prefix, static_cast<uint64_t>(V),
                         static_cast<uint32_t>(pk_sort_tile()), static_cast<uint32_t>(sort_tile(4)),
                         static_cast<const uint32_t*>(plan), L.D, static_cast<const uint32_t*>(d_status), gate));
        RMX_CHECK(cudaGetLastError());
        return RMX_OK;
    };
    if ((rc = launch_soup(nullptr))) return rc;
    // window mode (rmx_window.cuh): u32 keys of four passes sort by their top 16 bits only (decided
    // once the key layout is final: after the value-rank tables, before k_pack)
    // (D <= 3, like the speculative plans: C3's D = 4 tets -- 24 copies per vertex, windows of
    // ~2.5K rows -- measured 4.62 ms with it vs 4.63 without, C2 5.78 vs 6.90)
    const int win_ok = (sc == nullptr && win_enabled() && !ds2_enabled() && L.D <= 3) ? 1 : 0;
    if ((rc = rec.mark())) return rc;
    // ---- packed keys (packed mode)
    uint16_t* rank16 = reinterpret_cast<uint16_t*>(base + L.rank16);
    uint16_t* vinv = reinterpret_cast<uint16_t*>(base + L.vinv);
    uint32_t* spec = reinterpret_cast<uint32_t*>(base + L.spec);
    // rank tables and the new key layout (exact plan, value sets of the full pass); fallback = 1:
    // the same after a failed speculative plan (each kernel exits unless kSpecMiss)
    auto finish_value_plan = [&](int fallback) -> int {
        uint32_t* vstate = reinterpret_cast<uint32_t*>(base + L.vstate);
        // second chance when a row fell outside the sample: value sets again with the exact packing
        RMX_CHECK(launch(k_vsets_reset, 1, kBlock, 0, s, vsets, static_cast<uint32_t>(L.D * kValueWords), vstate,
                         static_cast<const uint32_t*>(gplan), static_cast<const uint32_t*>(vary),
                         static_cast<const uint32_t*>(svary), static_cast<const uint32_t*>(fields),
                         static_cast<const uint32_t*>(sfields), L.D, static_cast<const uint32_t*>(d_status),
                         static_cast<const uint32_t*>(fallback ? spec : nullptr)));
        ValueSetArgs ra{vtx, flags, idx, plan, fields, vsets, nullptr, vstate, d_status, static_cast<uint32_t>(V),
                        0u, vec, 1, gplan, 0, spec, fallback};
        int rc2 = dispatch_valueset(ra, L.D, s);
        if (rc2) return rc2;
        ValuePlanArgs pa{plan, vsets, nullptr, rank16, vinv, d_status, L.D, 1, vstate, gplan, svary, sfields, vary,
                         fields, spec, vstate, 0, fallback};
        RMX_CHECK(launch(k_value_plan, 1, 1024, 0, s, pa));
        RMX_CHECK(cudaGetLastError());
        return RMX_OK;
    };
    if (value_ranks && (rc = finish_value_plan(0))) return rc;
    uint8_t* dig = reinterpret_cast<uint8_t*>(base + L.pk_digits);
    const size_t dig_stride = align_up(static_cast<size_t>(V) + 16);
    {
        RMX_CHECK(launch(k_win_decide, 1, 32, 0, s, plan, L.D, win_ok, static_cast<const uint32_t*>(d_status),
                         static_cast<const uint32_t*>(nullptr), static_cast<const uint32_t*>(soup), win_rows,
                         static_cast<uint32_t>(V)));
        PackArgs a{vtx, flags, idx, plan, rows0, L.vals_off, dig, fields, rank16, d_status, static_cast<uint32_t>(V),
                   L.D, vec, vary, spec, 0, win_rows};
        if ((rc = dispatch_pack(a, s, value_ranks && spec_enabled() && L.D <= 3))) return rc;
        if (value_ranks) {
            // a speculative plan that k_pack's check failed (kSpecMiss): the path it skipped --
            // full value-set pass with its check, decision, K1a, plan, second chance, rank tables --
            // and the keys again (each kernel exits at once otherwise)
            uint32_t* vstate = reinterpret_cast<uint32_t*>(base + L.vstate);
            RMX_CHECK(launch(k_spec_reset, 1, 256, 0, s, static_cast<const uint32_t*>(spec), vary, fields, vsets,
                             vstate, L.D, static_cast<const uint32_t*>(d_status)));
            ValueSetArgs fv{vtx, flags, idx, gplan, sfields, vsets, svary, vstate, d_status,
                            static_cast<uint32_t>(V), 0u, vec, 0, gplan, 0, spec, 1};
            if ((rc = dispatch_valueset(fv, L.D, s))) return rc;
            ValuePlanArgs fd{gplan, vsets, nullptr, nullptr, nullptr, d_status, L.D, 0, nullptr, nullptr, nullptr,
                             nullptr, nullptr, nullptr, spec, vstate, 0, 1};
            RMX_CHECK(launch(k_value_plan, 1, 1024, 0, s, fd));
            VaryArgs fb{vtx, flags, idx, vary, fields, d_status, static_cast<uint32_t>(V), L.D, vec, 0u,
                        vstate, svary, sfields, spec};
            if ((rc = dispatch_vary(fb, s))) return rc;
            RMX_CHECK(launch(k_plan, 1, 32, 0, s, vary, fields, plan, L.D, d_status, hash_ok ? 1 : 0,
                             static_cast<const uint32_t*>(spec)));
            if ((rc = launch_soup(spec))) return rc;
            if ((rc = finish_value_plan(1))) return rc;
            RMX_CHECK(launch(k_win_decide, 1, 32, 0, s, plan, L.D, win_ok, static_cast<const uint32_t*>(d_status),
                             static_cast<const uint32_t*>(spec), static_cast<const uint32_t*>(soup), win_rows,
                             static_cast<uint32_t>(V)));
            a.fallback = 1;
            if ((rc = dispatch_pack(a, s))) return rc;
        }
    }
    if ((rc = rec.mark())) return rc;
    uint32_t* repl = reinterpret_cast<uint32_t*>(base + L.repl);
    if (lean) {  // packed keys only; keep the replacement row (k_unpack_pk reads it after the vertices are gone)
        RMX_CHECK(launch(k_lean_prepare, 1, 32, 0, s, static_cast<const uint32_t*>(plan), vtx, idx, repl, L.D,
                         d_status));
        RMX_CHECK(cudaGetLastError());
    }
    // ---- AoS rows of the whole vertex set (AoS mode only).  With D <= 2 at most 64 bits vary,
    // which the packed key always holds (plan_body: every run is >= 1 bit, so <= 64 runs): no AoS
    // kernels then (their stage events are still recorded).
    const bool aos = aos_possible(L.D) && !lean;
    if (aos) {
        BuildArgs a{vtx, flags, idx, rows0, hist, plan, d_status, static_cast<uint32_t>(V), L.D, vec};
        if ((rc = dispatch_build(a, s))) return rc;
    }
    HashArgs ha{vtx, flags, idx, plan, rows0, rows1, reinterpret_cast<uint32_t*>(base + L.hhist),
                reinterpret_cast<uint2*>(base + L.ukeys), reinterpret_cast<uint32_t*>(base + L.n_cand), hist,
                reinterpret_cast<const uint32_t*>(base + L.rank_of), d_status, static_cast<uint32_t>(V),
                L.ntiles_hash, L.D, vec, hash_raw};
    if (hash_ok && (rc = dispatch_hash_build(ha, s))) return rc;
    if ((rc = rec.mark())) return rc;
    for (int p = 0; p < kMaxPackedPasses; ++p) {
        if (p >= packed_passes_max(L.D)) {  // a packed key of D = 1 words has at most 4 digits
            if ((rc = rec.mark())) return rc;
            continue;
        }
        SortPkArgs a{rows0, rows1, L.vals_off, plan, reinterpret_cast<uint32_t*>(base + L.pk_counts),
                     reinterpret_cast<uint32_t*>(base + L.pk_totals), dig + (p & 1) * dig_stride,
                     dig + ((p + 1) & 1) * dig_stride, d_status, static_cast<uint32_t>(V), L.ntiles_pk, L.pk_cstride,
                     L.D, p, rank_force(), soup, soup_prefix, flags, 0, win_rows,
                     static_cast<uint32_t>(pk_sort_tile())};
        if ((rc = launch_sort_pk(a, s))) return rc;
        if ((rc = rec.mark())) return rc;
    }
    // ---- hash mode: candidate groups of the hash-sorted rows, one AoS row per group
    if (hash_ok) {
        SortArgs hs{rows0, rows1, plan, reinterpret_cast<uint32_t*>(base + L.hhist), desc,
                    reinterpret_cast<uint32_t*>(base + L.hcounters), d_status, static_cast<uint32_t>(V), L.ntiles, L.D,
                    0, rank_force(), nullptr, vtx, flags, idx, soup, soup_prefix};
        if ((rc = launch_hash_groups(ha, hs, s))) return rc;
    }
    if ((rc = rec.mark())) return rc;
    // ---- exact AoS sort: the whole vertex set (AoS mode) or the candidate rows (hash mode)
    const uint32_t* n_cand = reinterpret_cast<const uint32_t*>(base + L.n_cand);
    if (aos) {
        HistArgs a{rows0, rows1, hist, plan, d_status, static_cast<uint32_t>(V), L.D, n_cand};
        int grid = 0;
        rc = grid_for_stream(V, grid);
        if (rc) return rc;
        RMX_CHECK(launch(k_first_hist, grid, kBlock, 0, s, a));
        RMX_CHECK(cudaGetLastError());
    }
    if ((rc = rec.mark())) return rc;
    for (int p = 0; p < L.P; ++p) {  // K2 onesweep passes, least significant digit first
        if (aos) {
            SortArgs a{rows0, rows1, plan, hist, desc, counters, d_status, static_cast<uint32_t>(V), L.ntiles, L.D,
                       p, rank_force(), n_cand};
            if ((rc = dispatch_pass(a, s))) return rc;
        }
        if ((rc = rec.mark())) return rc;
    }
    // ---- K3 unique + bucketed pairs (AoS / hash, or packed), K3b map fill
    uint32_t* fill = reinterpret_cast<uint32_t*>(base + L.fill);
    if (aos) {
        UniqueArgs a{rows0, rows1, plan, desc3, counters + L.P, fill, d_status,
                     out_vtx, reinterpret_cast<unsigned long long*>(d_count),
                     sc ? sc->org_id : nullptr, sc ? sc->nodup : nullptr, sc ? sc->new_idx : nullptr,
                     sc ? sc->perm : nullptr, static_cast<uint32_t>(V), L.ntiles3, L.D, L.bucket_shift, n_cand};
        if ((rc = dispatch_unique(a, s))) return rc;
    }
    if ((rc = rec.mark())) return rc;
    {  // window mode: bounds (+ the fallback decision), the per-window unique kernel
        WinArgs wa{plan, rows0, rows0 + L.vals_off, reinterpret_cast<uint2*>(rows1),
                   reinterpret_cast<uint32_t*>(base + L.wstart), reinterpret_cast<uint32_t*>(base + L.wend),
                   reinterpret_cast<uint64_t*>(base + L.win_desc), reinterpret_cast<uint32_t*>(base + L.win_counter),
                   fill, reinterpret_cast<uint32_t*>(base + L.ukeys), reinterpret_cast<unsigned long long*>(d_count),
                   plan, d_status, static_cast<uint32_t>(V), L.D, L.bucket_shift, win_rows, static_cast<uint32_t>(V),
                   static_cast<const uint32_t*>(soup)};
        int g = 0;
        if ((rc = grid_for_stream((V + 7) / 8, g))) return rc;
        RMX_CHECK(launch(k_win_bounds, g, kBlock, 0, s, wa));
        if ((rc = grid_for_stream(V, g))) return rc;
        int gu = 0;
        if ((rc = persistent_grid(k_win_unique, WinSmem::bytes(), kWinCount, gu, kWinThreads))) return rc;
        RMX_CHECK(launch(k_win_unique, gu, kWinThreads, WinSmem::bytes(), s, wa));
        RMX_CHECK(cudaGetLastError());
        if ((rc = rec.mark())) return rc;  // (stage "window")
        // fallback (a window of more than kWinMaxRows rows): digit 0, the four passes, then the
        // usual unique kernels below
        RMX_CHECK(launch(k_win_digit0, g, kBlock, 0, s, static_cast<const uint32_t*>(plan), L.D, rows0,
                         static_cast<const uint32_t*>(rows0 + L.vals_off), dig, static_cast<const uint32_t*>(win_rows),
                         static_cast<const uint32_t*>(soup), static_cast<const uint32_t*>(d_status)));
        for (int p = 0; p < 4; ++p) {
            SortPkArgs fa{rows0, rows1, L.vals_off, plan, reinterpret_cast<uint32_t*>(base + L.pk_counts),
                          reinterpret_cast<uint32_t*>(base + L.pk_totals), dig + (p & 1) * dig_stride,
                          dig + ((p + 1) & 1) * dig_stride, d_status, static_cast<uint32_t>(V), L.ntiles_pk,
                          L.pk_cstride, L.D, p, rank_force(), soup, soup_prefix, flags, 1, win_rows,
                          static_cast<uint32_t>(pk_sort_tile())};
            if ((rc = launch_sort_pk(fa, s))) return rc;
        }
    }
    {
        uint32_t* counts = reinterpret_cast<uint32_t*>(base + L.tile_counts);
        HeadCountArgs h{rows0, rows1, plan, counts, d_status, static_cast<uint32_t>(V), L.ntiles3_pk,
                        static_cast<uint32_t>(kPkUniqTile), L.D, win_rows};
        int grid = 0;
        if ((rc = grid_for_stream(static_cast<uint64_t>(L.ntiles3_pk) * kBlock, grid))) return rc;
        RMX_CHECK(launch(k_head_count_pk, grid, kBlock, 0, s, h));
        RMX_CHECK(cudaGetLastError());
        RMX_CHECK(launch(k_tile_scan, 1, 1024, 0, s, counts, L.ntiles3_pk, plan, L.D,
                         reinterpret_cast<unsigned long long*>(d_count), d_status,
                         static_cast<const uint32_t*>(win_rows), static_cast<uint32_t>(kPkUniqTile)));
        RMX_CHECK(cudaGetLastError());
        void* ukeys = base + L.ukeys;
        UniquePkArgs a{rows0, rows1, L.vals_off, plan, counts, fill, d_status, ukeys,
                       sc ? sc->org_id : nullptr, sc ? sc->nodup : nullptr, sc ? sc->new_idx : nullptr,
                       sc ? sc->perm : nullptr, static_cast<uint32_t>(V), L.ntiles3_pk, L.D, L.bucket_shift, win_rows,
                       static_cast<uint32_t>(V)};
        if ((rc = launch_unique_pk(a, s))) return rc;
        // lean: the unique rows go to the final sort buffer (read completely by k_unique_pk by then)
        UnpackPkArgs u{plan, lean ? repl : vtx, lean ? repl + RMX_MAX_DIM : idx, vary, fields, ukeys, vinv,
                       out_vtx, reinterpret_cast<unsigned long long*>(d_count), d_status, L.D,
                       (lean || aligned16(out_vtx)) ? 1 : 0, lean ? rows0 : nullptr, lean ? rows1 : nullptr,
                       d_where};
        if ((rc = launch_unpack_pk(u, V, s))) return rc;
    }
    if ((rc = rec.mark())) return rc;
    {
        if (hash_ok) {  // rank_of[candidate] from the candidates' pairs, then (origin, new index) pairs
            int grid = 0;
            if ((rc = grid_for_stream((V + 1) / 2, grid))) return rc;
            RMX_CHECK(launch(k_map_fill, grid, kBlock, 0, s, static_cast<const uint32_t*>(plan),
                             static_cast<const uint32_t*>(rows0), static_cast<const uint32_t*>(rows1),
                             reinterpret_cast<uint32_t*>(base + L.rank_of), static_cast<uint32_t>(V),
                             static_cast<const uint32_t*>(d_status), L.D, 2, n_cand,
                             static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                             static_cast<const uint32_t*>(nullptr), 0));
            RMX_CHECK(cudaGetLastError());
            int gp = 0;
            if ((rc = persistent_grid(k_hash_pairs, 0, (V + kPairsTile - 1) / kPairsTile, gp))) return rc;
            RMX_CHECK(launch(k_hash_pairs, gp, kBlock, 0, s, ha, reinterpret_cast<uint32_t*>(base + L.fill2),
                             L.bucket_shift));
            RMX_CHECK(cudaGetLastError());
        }
        const uint64_t threads = (V + 1) / 2;
        RMX_CHECK(launch(k_map_fill, static_cast<unsigned>((threads + kBlock - 1) / kBlock), kBlock, 0, s,
                         static_cast<const uint32_t*>(plan), static_cast<const uint32_t*>(rows0),
                         static_cast<const uint32_t*>(rows1), map, static_cast<uint32_t>(V),
                         static_cast<const uint32_t*>(d_status), L.D, 0, n_cand, static_cast<const uint32_t*>(soup),
                         out_idx, static_cast<const uint32_t*>(fill), L.bucket_shift));
        RMX_CHECK(cudaGetLastError());
    }
    if ((rc = rec.mark())) return rc;
    // K4 remap
    {
        RemapArgs a{idx, map, out_idx, I, d_status, (aligned16(idx) && aligned16(out_idx)) ? 1 : 0, soup};
        int grid = 0;
        rc = grid_for_stream(a.vec ? (I + 3) / 4 : I, grid);
        if (rc) return rc;
        RMX_CHECK(launch(k_remap, grid, kBlock, 0, s, a));
        RMX_CHECK(cudaGetLastError());
    }
    return rec.mark();
}

}  // namespace

extern "C" {

const char* rmx_version(void) { return "paper_2109_09812_b200 0.1.0 (sm_100a)"; }

const char* rmx_strerror(int code) {
    switch (code) {
        case RMX_OK: return "ok";
        case RMX_EINVAL: return g_err[0] ? g_err : "invalid argument";
        case RMX_ERANGE: return g_err[0] ? g_err : "vertex count exceeds 32-bit index range";
        case RMX_ECUDA: return g_err[0] ? g_err : "CUDA error";
        case RMX_ENOSPC: return g_err[0] ? g_err : "workspace too small";
        default: return "unknown error";
    }
}

size_t rmx_workspace_bytes(uint64_t n_vertices, uint32_t dim, uint64_t n_elements, uint32_t arity) {
    (void)n_elements;
    (void)arity;
    if (dim < 1 || dim > RMX_MAX_DIM) return 0;
    return make_layout(n_vertices, dim).total;
}

int rmx_reindex(const uint32_t* vtx_bits, uint64_t n_vertices, uint32_t dim, const uint32_t* idx,
                uint64_t n_elements, uint32_t arity, uint32_t* out_vtx_bits, uint32_t* out_idx,
                uint64_t* d_new_count, uint32_t* d_status, void* workspace, size_t workspace_bytes,
                const rmx_scratch* scratch, void* stream) {
    return run_pipeline(vtx_bits, n_vertices, dim, idx, n_elements, arity, out_vtx_bits, out_idx, d_new_count,
                        d_status, workspace, workspace_bytes, scratch, static_cast<cudaStream_t>(stream), nullptr,
                        0);
}

size_t rmx_lean_workspace_bytes(uint64_t n_vertices, uint32_t dim, uint64_t n_elements, uint32_t arity) {
    (void)n_elements;
    (void)arity;
    if (dim < 3 || dim > RMX_MAX_DIM) return 0;
    return make_layout(n_vertices, dim, true).total;
}

size_t rmx_lean_result_offset(uint64_t n_vertices, uint32_t dim) {
    if (dim < 3 || dim > RMX_MAX_DIM) return 0;
    return make_layout(n_vertices, dim, true).rows0;
}

int rmx_reindex_lean(uint32_t* vtx_bits, uint64_t n_vertices, uint32_t dim, const uint32_t* idx,
                     uint64_t n_elements, uint32_t arity, uint32_t* out_idx, uint64_t* d_new_count,
                     uint32_t* d_status, uint32_t* d_where, void* workspace, size_t workspace_bytes,
                     void* stream) {
    return run_pipeline(vtx_bits, n_vertices, dim, idx, n_elements, arity, nullptr, out_idx, d_new_count, d_status,
                        workspace, workspace_bytes, nullptr, static_cast<cudaStream_t>(stream), nullptr, 0, true,
                        d_where);
}

int rmx_reindex_profiled(const uint32_t* vtx_bits, uint64_t n_vertices, uint32_t dim, const uint32_t* idx,
                         uint64_t n_elements, uint32_t arity, uint32_t* out_vtx_bits, uint32_t* out_idx,
                         uint64_t* d_new_count, uint32_t* d_status, void* workspace, size_t workspace_bytes,
                         const rmx_scratch* scratch, void* stream, void* const* events, int n_events) {
    return run_pipeline(vtx_bits, n_vertices, dim, idx, n_elements, arity, out_vtx_bits, out_idx, d_new_count,
                        d_status, workspace, workspace_bytes, scratch, static_cast<cudaStream_t>(stream), events,
                        n_events);
}

struct rmx_graph {
    cudaGraphExec_t exec;
};

int rmx_graph_create(const uint32_t* vtx_bits, uint64_t n_vertices, uint32_t dim, const uint32_t* idx,
                     uint64_t n_elements, uint32_t arity, uint32_t* out_vtx_bits, uint32_t* out_idx,
                     uint64_t* d_new_count, uint32_t* d_status, void* workspace, size_t workspace_bytes,
                     const rmx_scratch* scratch, rmx_graph** out) {
    if (!out) return RMX_EINVAL;
    *out = nullptr;
    if (dim < 1 || dim > RMX_MAX_DIM) {
        std::snprintf(g_err, sizeof(g_err), "dim %u outside [1, %d]", dim, RMX_MAX_DIM);
        return RMX_EINVAL;
    }
    cudaStream_t cs = nullptr;
    cudaGraph_t cg = nullptr;
    RMX_CHECK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    int rc = RMX_OK;
    bool capturing = false;
    if (cudaStreamBeginCapture(cs, kCaptureMode) == cudaSuccess) {
        capturing = true;
        rc = run_pipeline(vtx_bits, n_vertices, dim, idx, n_elements, arity, out_vtx_bits, out_idx, d_new_count,
                          d_status, workspace, workspace_bytes, scratch, cs, nullptr, 0);
    } else {
        rc = RMX_ECUDA;
    }
    if (capturing && cudaStreamEndCapture(cs, &cg) != cudaSuccess && rc == RMX_OK) rc = RMX_ECUDA;
    cudaGraphExec_t exec = nullptr;
    if (rc == RMX_OK) {
        const cudaError_t e = cudaGraphInstantiate(&exec, cg, 0);
        if (e != cudaSuccess) {
            std::snprintf(g_err, sizeof(g_err), "graph instantiate: %s", cudaGetErrorString(e));
            rc = RMX_ECUDA;
        }
    }
    (void)cudaGetLastError();
    if (cg) cudaGraphDestroy(cg);
    cudaStreamDestroy(cs);
    if (rc != RMX_OK) return rc;
    *out = new rmx_graph{exec};
    return RMX_OK;
}

int rmx_graph_launch(rmx_graph* graph, void* stream) {
    if (!graph) return RMX_EINVAL;
    RMX_CHECK(cudaGraphLaunch(graph->exec, static_cast<cudaStream_t>(stream)));
    return RMX_OK;
}

void rmx_graph_destroy(rmx_graph* graph) {
    if (!graph) return;
    cudaGraphExecDestroy(graph->exec);
    delete graph;
}

int rmx_kernel_launches(uint32_t dim) {
    // mark + expand, vary, plan, [D >= 3: build_rows], pack,
    // [dim <= kMaxRankDim, meshes of >= 2^25 rows (value_rank_min_rows): K1a over a sample, guessed plan,
    //  value-set sample x 2, value plan, value sets + K1a check in one pass, value plan, second-chance
    //  reset + value sets + value plan (exit unless a row fell outside the sample)],
    // packed_passes_max x (upsweep, colscan, downsweep),
    // [3 <= D <= kHashMaxDim, no scratch: hash build, 2 hashed passes, dedup, rank map fill, pairs],
    // [D >= 3: first_hist, 4 D AoS passes, unique (AoS)],
    // head_count + tile_scan + unique_pk + unpack_pk, map_fill, remap
    const int value_ranks = (dim <= static_cast<uint32_t>(kMaxRankDim) && value_rank_enabled()) ? 10 : 0;
    const int D = static_cast<int>(dim);
    const int aos = aos_possible(D) ? 1 + 1 + 4 * D + 1 : 0;
    const int hash = (hash_possible(D) && hash_enabled()) ? 6 : 0;
    return 4 + value_ranks + 1 + 3 * packed_passes_max(D) + aos + hash + 4 + 2;
}

unsigned long long rmx_kernel_launches_total(void) { return g_launches.load(std::memory_order_relaxed); }

int rmx_debug_oob_count(unsigned long long* out) {
#ifdef RMX_CHECKED
    if (!out) return RMX_EINVAL;
    RMX_CHECK(cudaDeviceSynchronize());
    RMX_CHECK(cudaMemcpyFromSymbol(out, g_rmx_oob, sizeof(*out)));
    return RMX_OK;
#else
    (void)out;
    return RMX_EINVAL;  // not a checked build
#endif
}

int rmx_stage_count(uint32_t dim) { return static_cast<int>(4 * dim) + 6 + kMaxPackedPasses + 2 + 5; }

const char* rmx_stage_name(uint32_t dim, int k) {
    static thread_local char buf[32];
    const int P = static_cast<int>(4 * dim);
    static const char* head[] = {"start", "mark", "vary", "plan", "pack", "build_rows"};
    if (k >= 0 && k < 6) return head[k];
    k -= 6;
    if (k < kMaxPackedPasses) {
        std::snprintf(buf, sizeof(buf), "pk_pass_%d", k);
        return buf;
    }
    k -= kMaxPackedPasses;
    if (k == 0) return "hash_groups";
    if (k == 1) return "first_hist";
    k -= 2;
    if (k < P) {
        std::snprintf(buf, sizeof(buf), "sort_pass_%d", k);
        return buf;
    }
    k -= P;
    static const char* tail[] = {"unique", "window", "unique_pk", "map_fill", "remap"};
    if (k >= 0 && k < 5) return tail[k];
    return "";
}

int rmx_plan_info(void* workspace, uint64_t n_vertices, uint32_t dim, void* stream, uint32_t* info) {
    if (!workspace || !info || dim < 1 || dim > RMX_MAX_DIM) return RMX_EINVAL;
    const Layout L = make_layout(n_vertices, dim);
    uint32_t h[8] = {0};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    char* plan = static_cast<char*>(workspace) + L.plan;
    RMX_CHECK(cudaMemcpyAsync(h, plan, 8, cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaMemcpyAsync(h + 2, plan + pk_base(L.P) * 4, 16, cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaStreamSynchronize(s));
    info[0] = h[2];  // mode: 0 AoS rows, 1 packed keys, 2 hash (rmx_hash.cuh)
    info[1] = h[2] ? h[3] : 0u;  // key words
    info[2] = h[2] ? h[4] : 0u;  // varying bits
    info[3] = h[2] == 1u ? h[5] : h[1];  // executed sort passes (hash mode: of the candidate rows)
    return RMX_OK;
}

int rmx_plan_key_info(void* workspace, uint64_t n_vertices, uint32_t dim, void* stream, uint32_t* info) {
    if (!workspace || !info || dim < 1 || dim > RMX_MAX_DIM) return RMX_EINVAL;
    const Layout L = make_layout(n_vertices, dim);
    uint32_t pk[8] = {0}, rk[RMX_MAX_DIM] = {0}, vb[4 + 4 * kMaxRankDim] = {0};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const char* plan = static_cast<const char*>(workspace) + L.plan;
    RMX_CHECK(cudaMemcpyAsync(pk, plan + pk_base(L.P) * 4, sizeof(pk), cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaMemcpyAsync(rk, plan + pk_rank_base(L.P) * 4, sizeof(rk), cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaMemcpyAsync(vb, plan + pk_value_base(L.P) * 4, sizeof(vb), cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaStreamSynchronize(s));
    for (int k = 0; k < 4; ++k) info[k] = 0u;
    if (!pk[0]) return RMX_OK;
    uint32_t fmask = 0, plain = pk[2];
    for (int c = 0; c < L.D && c < 32; ++c)
        if (rk[c] >> 31) fmask |= 1u << c;
    const bool vr = L.D <= kMaxRankDim && vb[0] == 2u;
    if (vr) {
        plain = 0;
        for (int c = 0; c < L.D; ++c) plain += vb[4 + 4 * c + 1];
    }
    info[0] = fmask;                // components whose sign+exponent field is ranked
    info[1] = vr ? vb[1] : 0u;      // components replaced by their value rank
    info[2] = plain;                // key bits before value ranks
    info[3] = pk[2];                // key bits
    return RMX_OK;
}

int rmx_plan_guess_info(void* workspace, uint64_t n_vertices, uint32_t dim, void* stream, uint32_t* info) {
    if (!workspace || !info || dim < 1 || dim > RMX_MAX_DIM) return RMX_EINVAL;
    const Layout L = make_layout(n_vertices, dim);
    for (int k = 0; k < 4; ++k) info[k] = 0u;
    if (L.D > kMaxRankDim) return RMX_OK;
    uint32_t pk[8] = {0}, vb[2] = {0}, st = 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const char* base = static_cast<const char*>(workspace);
    RMX_CHECK(cudaMemcpyAsync(pk, base + L.gplan + pk_base(L.P) * 4, sizeof(pk), cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaMemcpyAsync(vb, base + L.gplan + pk_value_base(L.P) * 4, sizeof(vb), cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaMemcpyAsync(&st, base + L.vstate, 4, cudaMemcpyDeviceToHost, s));
    uint32_t sp = 0;
    RMX_CHECK(cudaMemcpyAsync(&sp, base + L.spec, 4, cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaStreamSynchronize(s));
    info[0] = pk[0] ? pk[2] : 0u;  // key bits of the plan guessed from the sample
    info[1] = vb[0];               // 1: value sets judged worth collecting
    info[2] = vb[1];               // candidate components
    info[3] = st | (sp << 8);      // kVstateChecked | kVstateMiss of the full pass; bit 8: the plan was
                                   // speculative (sample-saturated value sets), bit 9: k_pack's check failed
    return RMX_OK;
}

int rmx_hash_info(void* workspace, uint64_t n_vertices, uint32_t dim, void* stream, uint32_t* info) {
    if (!workspace || !info || dim < 1 || dim > RMX_MAX_DIM) return RMX_EINVAL;
    const Layout L = make_layout(n_vertices, dim);
    uint32_t pk0 = 0, nc = 0, pl[2] = {0, 0};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const char* base = static_cast<const char*>(workspace);
    RMX_CHECK(cudaMemcpyAsync(&pk0, base + L.plan + pk_base(L.P) * 4, 4, cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaMemcpyAsync(&nc, base + L.n_cand, 4, cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaMemcpyAsync(pl, base + L.plan, 8, cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaStreamSynchronize(s));
    const bool hash = pk0 == 2u;
    info[0] = hash ? 1u : 0u;                      // the call ran in hash mode
    info[1] = hash ? nc : 0u;                      // candidate rows (distinct keys per dedup tile)
    info[2] = hash ? pl[1] : 0u;                   // executed AoS passes over the candidates
    info[3] = static_cast<uint32_t>(kHashTile);    // rows per dedup tile
    return RMX_OK;
}

int rmx_window_info(void* workspace, uint64_t n_vertices, uint32_t dim, void* stream, uint32_t* info) {
    if (!workspace || !info || dim < 1 || dim > RMX_MAX_DIM) return RMX_EINVAL;
    const Layout L = make_layout(n_vertices, dim);
    uint32_t pk[8] = {0}, nd = 0;
    std::vector<uint32_t> ws(kWinCount), we(kWinCount);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const char* base = static_cast<const char*>(workspace);
    RMX_CHECK(cudaMemcpyAsync(pk, base + L.plan + pk_base(L.P) * 4, sizeof(pk), cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaMemcpyAsync(ws.data(), base + L.wstart, kWinCount * 4, cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaMemcpyAsync(we.data(), base + L.wend, kWinCount * 4, cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaMemcpyAsync(&nd, base + L.win_rows, 4, cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaStreamSynchronize(s));
    uint32_t nonempty = 0, maxrows = 0;
    for (uint32_t w = 0; w < kWinCount; ++w)
        if (ws[w] != 0xFFFFFFFFu) {
            ++nonempty;
            maxrows = std::max(maxrows, we[w] - ws[w]);
        }
    info[0] = pk[6] | (pk[7] << 1);  // bit 0 window mode decided, bit 1 its fallback ran
    info[1] = nd;                    // used rows sorted (unused rows dropped by the first pass)
    info[2] = nonempty;              // non-empty windows
    info[3] = maxrows;               // rows of the largest window
    return RMX_OK;
}

int rmx_soup_info(void* workspace, uint64_t n_vertices, uint32_t dim, void* stream, uint32_t* info) {
    if (!workspace || !info || dim < 1 || dim > RMX_MAX_DIM) return RMX_EINVAL;
    const Layout L = make_layout(n_vertices, dim);
    uint32_t soup = 0, order = 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const char* base = static_cast<const char*>(workspace);
    RMX_CHECK(cudaMemcpyAsync(&soup, base + L.soup, 4, cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaMemcpyAsync(&order, base + L.order, 4, cudaMemcpyDeviceToHost, s));
    RMX_CHECK(cudaStreamSynchronize(s));
    info[0] = soup;                    // soup mode: the index count I (0: off)
    info[1] = (order & 1u) ? 0u : 1u;  // the indices were strictly increasing
    return RMX_OK;
}

int rmx_last_executed_passes(void* workspace, uint64_t n_vertices, uint32_t dim, void* stream) {
    if (!workspace || dim < 1 || dim > RMX_MAX_DIM) return -1;
    const Layout L = make_layout(n_vertices, dim);
    uint32_t v = 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (cudaMemcpyAsync(&v, static_cast<char*>(workspace) + L.plan + 4, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return -1;
    if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
    return static_cast<int>(v);
}

int rmx_debug_phase_cycles(unsigned long long* out, int n, int reset) {
#ifdef RMX_PHASES
    unsigned long long h[4] = {0};
    RMX_CHECK(cudaMemcpyFromSymbol(h, g_lb_stats, sizeof(h)));
    for (int i = 0; i < n && i < 4; ++i) out[i] = h[i];
    if (reset) {
        unsigned long long z[4] = {0};
        RMX_CHECK(cudaMemcpyToSymbol(g_lb_stats, z, sizeof(z)));
    }
    return 4;
#else
    for (int i = 0; i < n; ++i) out[i] = 0;
    (void)reset;
    return 0;
#endif
}

int rmx_gather_u32(const uint32_t* table, uint64_t n_table, const uint32_t* idx, uint64_t n, uint32_t* out,
                   uint32_t* d_status, void* stream) {
    g_err[0] = '\0';
    if (n == 0) return RMX_OK;
    if (!table || !idx || !out || !d_status) return RMX_EINVAL;
    int grid = 0;
    int rc = grid_for_stream(n, grid);
    if (rc) return rc;
    k_gather<<<grid, kBlock, 0, static_cast<cudaStream_t>(stream)>>>(table, n_table, idx, n, out, d_status);
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

size_t rmx_select_workspace_bytes(uint64_t n_elements) {
    return static_cast<size_t>((n_elements + kKeepTile - 1) / kKeepTile) * 4 + 256;
}

int rmx_select_elements(const uint32_t* idx, uint64_t n_elements, uint32_t arity, const uint8_t* keep,
                        uint32_t* out_idx, uint64_t* d_kept, void* workspace, size_t workspace_bytes, void* stream) {
    g_err[0] = '\0';
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!d_kept || arity < 1) return RMX_EINVAL;
    RMX_CHECK(cudaMemsetAsync(d_kept, 0, sizeof(uint64_t), s));
    if (n_elements == 0) return RMX_OK;
    if (!idx || !keep || !out_idx) return RMX_EINVAL;
    if (n_elements >= (1ull << 32)) return RMX_ERANGE;
    if (!workspace || workspace_bytes < rmx_select_workspace_bytes(n_elements)) return RMX_ENOSPC;
    uint32_t* counts = static_cast<uint32_t*>(workspace);
    const uint32_t tiles = static_cast<uint32_t>((n_elements + kKeepTile - 1) / kKeepTile);
    k_keep_count<<<tiles, kBlock, 0, s>>>(keep, n_elements, counts);
    RMX_CHECK(cudaGetLastError());
    k_rows_scan<<<1, 1024, 0, s>>>(counts, tiles, reinterpret_cast<unsigned long long*>(d_kept));
    RMX_CHECK(cudaGetLastError());
    k_keep_compact<<<tiles, kBlock, 0, s>>>(idx, n_elements, arity, keep, counts, out_idx);
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

int rmx_offset_indices(const uint32_t* idx, uint64_t n, uint32_t offset, uint32_t* out, void* stream) {
    g_err[0] = '\0';
    if (n == 0) return RMX_OK;
    if (!idx || !out) return RMX_EINVAL;
    const int vec = (aligned16(idx) && aligned16(out)) ? 1 : 0;
    int grid = 0;
    int rc = grid_for_stream(vec ? (n + 3) / 4 : n, grid);
    if (rc) return rc;
    k_offset_indices<<<grid, kBlock, 0, static_cast<cudaStream_t>(stream)>>>(idx, n, offset, out, vec);
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

int rmx_scatter_rows(const uint32_t* src, uint64_t n, uint32_t words, const uint64_t* bounds, uint32_t groups,
                     const uint64_t* dst_ptrs, const uint64_t* dst_off, void* stream) {
    g_err[0] = '\0';
    if (n == 0) return RMX_OK;
    if (!src || !bounds || !dst_ptrs || !dst_off || words < 1 || groups < 1) return RMX_EINVAL;
    int grid = 0;
    int rc = grid_for_stream(n * words, grid);
    if (rc) return rc;
    k_scatter_rows<<<grid, kBlock, 0, static_cast<cudaStream_t>(stream)>>>(src, n, words, bounds, groups, dst_ptrs,
                                                                           dst_off);
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

size_t rmx_merge_workspace_bytes(uint64_t n_rows, uint32_t key_words) {
    const uint64_t W = static_cast<uint64_t>(key_words) + 1;
    const uint64_t tiles = (n_rows + kMergeTile - 1) / kMergeTile;
    // two row buffers (+64 words of slack each), tile counts (+64), up to 8 bytes of alignment
    // padding before the splits, the splits: the same layout rmx_merge_unique_runs carves
    return static_cast<size_t>(2 * (n_rows * W + 64) * 4 + (tiles + 64) * 4 + 8 + (tiles + 1) * 8 + 256);
}

int rmx_merge_unique_runs(const uint32_t* keys, uint64_t n_rows, uint32_t key_words, const uint64_t* run_starts,
                          uint32_t n_runs, uint32_t* out_keys, uint32_t* rank_of, uint64_t* d_count,
                          void* workspace, size_t workspace_bytes, void* stream) {
    g_err[0] = '\0';
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!d_count) return RMX_EINVAL;
    RMX_CHECK(cudaMemsetAsync(d_count, 0, sizeof(uint64_t), s));
    if (n_rows == 0) return RMX_OK;
    const uint32_t D = key_words, W = key_words + 1;
    if (!keys || !run_starts || !out_keys || !rank_of || D < 1 || W > kMergeMaxW || n_runs < 1 ||
        n_rows >= (1ull << 32)) {
        std::snprintf(g_err, sizeof(g_err), "merge: bad arguments (key words %u, runs %u)", key_words, n_runs);
        return RMX_EINVAL;
    }
    if (!workspace || workspace_bytes < rmx_merge_workspace_bytes(n_rows, key_words)) return RMX_ENOSPC;
    uint32_t* buf[2] = {static_cast<uint32_t*>(workspace),
                        static_cast<uint32_t*>(workspace) + n_rows * W + 64};
    uint32_t* counts = buf[1] + n_rows * W + 64;
    const uint64_t max_tiles = (n_rows + kMergeTile - 1) / kMergeTile;
    uint64_t* splits = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(counts + max_tiles + 64) + 7) & ~static_cast<uintptr_t>(7));
    int rc = RMX_OK;
    int grid = 0;
    if ((rc = grid_for_stream(n_rows, grid))) return rc;
    // pairwise rounds: runs (0,1), (2,3), ... until one run is left; the first round reads the
    // keys themselves (rows get their arrival position as they are staged)
    std::vector<uint64_t> starts(run_starts, run_starts + n_runs);
    starts.push_back(n_rows);
    const size_t smem = 2 * (static_cast<size_t>(kMergeTile) * W + kMergeTile / 8 + 1) * 4;  // padded in + out
    switch (W) {
#define RMX_SMEM_W(w)                                                \
    case w:                                                          \
        if ((rc = ensure_smem(k_merge_path<w, true>, smem))) break;  \
        rc = ensure_smem(k_merge_path<w, false>, smem);              \
        break;
        RMX_SMEM_W(2) RMX_SMEM_W(3) RMX_SMEM_W(4) RMX_SMEM_W(5) RMX_SMEM_W(6) RMX_SMEM_W(7) RMX_SMEM_W(8)
        RMX_SMEM_W(9)
#undef RMX_SMEM_W
    }
    if (rc) return rc;
    auto to_rows = [&](uint64_t a0, uint64_t n, uint32_t* dst) -> int {  // keys -> rows (odd run, 1 run)
        switch (W) {
#define RMX_INIT_W(w)                                                                                 \
    case w: k_merge_rows_init<w><<<grid, kBlock, 0, s>>>(keys + a0 * D, n, static_cast<uint32_t>(a0), dst); \
        break;
            RMX_INIT_W(2) RMX_INIT_W(3) RMX_INIT_W(4) RMX_INIT_W(5) RMX_INIT_W(6) RMX_INIT_W(7) RMX_INIT_W(8)
            RMX_INIT_W(9)
#undef RMX_INIT_W
        }
        RMX_CHECK(cudaGetLastError());
        return RMX_OK;
    };
    int cur = 0;
    bool first = true;
    if (starts.size() == 2) {  // one run: rows straight from the keys
        if ((rc = to_rows(0, n_rows, buf[0]))) return rc;
        first = false;
    }
    while (starts.size() > 2) {
        std::vector<uint64_t> next;
        for (size_t r = 0; r + 1 < starts.size(); r += 2) {
            const uint64_t a0 = starts[r], a1 = starts[r + 1];
            const uint64_t b1 = (r + 2 < starts.size()) ? starts[r + 2] : a1;
            next.push_back(a0);
            const uint64_t n = b1 - a0;
            if (r + 2 >= starts.size() || n == 0) {  // odd run out: carried to the next round
                if (n) {
                    if (first) {
                        if ((rc = to_rows(a0, n, buf[cur ^ 1] + a0 * W))) return rc;
                    } else {
                        RMX_CHECK(cudaMemcpyAsync(buf[cur ^ 1] + a0 * W, buf[cur] + a0 * W, n * W * 4,
                                                  cudaMemcpyDeviceToDevice, s));
                    }
                }
                continue;
            }
            const unsigned blocks = static_cast<unsigned>((n + kMergeTile - 1) / kMergeTile);
            const uint32_t S = first ? D : W;
            const uint32_t* src = first ? keys : buf[cur];
            const uint32_t* A = src + a0 * S;
            const uint32_t* B = src + a1 * S;
            uint32_t* O = buf[cur ^ 1] + a0 * W;
            k_merge_splits<<<(blocks + 1 + kBlock - 1) / kBlock, kBlock, 0, s>>>(A, a1 - a0, B, b1 - a1, S, D, splits,
                                                                                 blocks + 1);
            RMX_CHECK(cudaGetLastError());
            const uint32_t ao = static_cast<uint32_t>(a0), bo = static_cast<uint32_t>(a1);
            switch (W * 2 + (first ? 1 : 0)) {
#define RMX_MERGE_W(w)                                                                                          \
    case 2 * w: k_merge_path<w, false><<<blocks, kBlock, smem, s>>>(A, a1 - a0, B, b1 - a1, ao, bo, splits, O); \
        break;                                                                                                  \
    case 2 * w + 1: k_merge_path<w, true><<<blocks, kBlock, smem, s>>>(A, a1 - a0, B, b1 - a1, ao, bo, splits, O); \
        break;
                RMX_MERGE_W(2) RMX_MERGE_W(3) RMX_MERGE_W(4) RMX_MERGE_W(5) RMX_MERGE_W(6) RMX_MERGE_W(7)
                RMX_MERGE_W(8) RMX_MERGE_W(9)
#undef RMX_MERGE_W
            }
            RMX_CHECK(cudaGetLastError());
        }
        next.push_back(n_rows);
        starts.swap(next);
        cur ^= 1;
        first = false;
    }
    const uint32_t tiles = static_cast<uint32_t>((n_rows + kMergeTile - 1) / kMergeTile);
    k_rows_heads<<<tiles, kBlock, 0, s>>>(buf[cur], n_rows, W, D, counts);
    RMX_CHECK(cudaGetLastError());
    k_rows_scan<<<1, 1024, 0, s>>>(counts, tiles, reinterpret_cast<unsigned long long*>(d_count));
    RMX_CHECK(cudaGetLastError());
    k_rows_unique<<<tiles, kBlock, 0, s>>>(buf[cur], n_rows, W, D, counts, out_keys, rank_of);
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

int rmx_welded_tile_sizes(uint32_t n, uint64_t* n_vertices, uint64_t* n_elements) {
    if (n < 1) return RMX_EINVAL;
    const uint64_t pts = static_cast<uint64_t>(n + 1) * (n + 1);
    if (n_vertices) *n_vertices = pts + pts / 20;
    if (n_elements) *n_elements = 2ull * n * n;
    return RMX_OK;
}

int rmx_gen_welded_tile(uint32_t n, uint32_t row0, uint64_t seed, int shuffle, uint32_t* out_vtx_bits,
                        uint32_t* out_idx, void* stream) {
    if (n < 1 || !out_vtx_bits || !out_idx) return RMX_EINVAL;
    TileArgs a{};
    a.n = n;
    a.row0 = row0;
    a.shuffle = shuffle ? 1 : 0;
    a.n_pts = static_cast<uint64_t>(n + 1) * (n + 1);
    a.n_unused = a.n_pts / 20;
    a.n_elem = 2ull * n * n;
    if (a.n_pts + a.n_unused >= (1ull << 32)) return RMX_ERANGE;
    a.pts = make_perm(a.n_pts, seed);
    a.elems = make_perm(a.n_elem, seed + 1);
    a.useed = splitmix64(seed + 0x5555);
    a.vtx = out_vtx_bits;
    a.idx = out_idx;
    int grid = 0;
    int rc = grid_for_stream(a.n_elem, grid);
    if (rc) return rc;
    k_gen_welded_tile<<<grid, kBlock, 0, static_cast<cudaStream_t>(stream)>>>(a);
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

int rmx_lower_bound_rows(const uint32_t* rows, uint64_t n, uint32_t dim, const uint32_t* queries, uint64_t n_queries,
                         uint64_t* out_positions, void* stream) {
    g_err[0] = '\0';
    if (n_queries == 0) return RMX_OK;
    if (dim < 1 || !queries || !out_positions || (n && !rows)) return RMX_EINVAL;
    const unsigned grid = static_cast<unsigned>((n_queries + 127) / 128);
    k_lower_bound<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(
        rows, n, static_cast<int>(dim), queries, n_queries, reinterpret_cast<unsigned long long*>(out_positions));
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

int rmx_lattice_sizes(int kind, uint32_t nx, uint32_t ny, uint32_t nz, uint64_t n_elem_take, uint64_t* n_elements,
                      uint64_t* n_vertices) {
    if (kind != 0 && kind != 1) return RMX_EINVAL;
    const uint64_t K = kind == 0 ? 3 : 4;
    const uint64_t E = kind == 0 ? 2ull * nx * ny : 6ull * nx * ny * nz;
    const uint64_t take = n_elem_take < E ? n_elem_take : E;
    const uint64_t n_unused = (E * K) / 20;
    if (n_elements) *n_elements = E;
    if (n_vertices) *n_vertices = take * K + (E ? (take * n_unused) / E : 0);
    return RMX_OK;
}

int rmx_gen_lattice_soup_range(int kind, uint32_t nx, uint32_t ny, uint32_t nz, uint64_t seed, uint64_t e_begin,
                               uint64_t e_end, uint32_t* out_vtx_bits, uint32_t* out_idx, void* stream) {
    if (kind != 0 && kind != 1) return RMX_EINVAL;
    GenArgs g{};
    g.kind = kind;
    g.nx = nx;
    g.ny = ny;
    g.nz = nz;
    const uint64_t K = kind == 0 ? 3 : 4;
    g.n_elem = kind == 0 ? 2ull * nx * ny : 6ull * nx * ny * nz;
    g.take = e_end < g.n_elem ? e_end : g.n_elem;
    g.e0 = e_begin < g.take ? e_begin : g.take;
    g.n_unused = (g.n_elem * K) / 20;
    g.v0 = g.e0 * K + (g.n_elem ? (g.e0 * g.n_unused) / g.n_elem : 0);
    if (g.take == g.e0) return RMX_OK;
    int bits = 0;
    while ((1ull << bits) < g.n_elem) ++bits;  // bit length of n-1
    if (bits < 2) bits = 2;
    bits += bits & 1;
    g.half = static_cast<uint32_t>(bits / 2);
    g.mask = (1ull << g.half) - 1;
    for (int r = 0; r < 4; ++r) g.keys[r] = splitmix64(static_cast<uint64_t>(r) + seed * 4 + 1);
    g.useed = splitmix64(seed + 0x5555);
    g.vtx = out_vtx_bits;
    g.idx = out_idx;
    int grid = 0;
    int rc = grid_for_stream(g.take - g.e0, grid);
    if (rc) return rc;
    k_gen_lattice<<<grid, kBlock, 0, static_cast<cudaStream_t>(stream)>>>(g);
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

int rmx_gen_lattice_soup(int kind, uint32_t nx, uint32_t ny, uint32_t nz, uint64_t seed, uint64_t n_elem_take,
                         uint32_t* out_vtx_bits, uint32_t* out_idx, void* stream) {
    return rmx_gen_lattice_soup_range(kind, nx, ny, nz, seed, 0, n_elem_take, out_vtx_bits, out_idx, stream);
}

int rmx_gen_grid_quads(uint32_t n, uint32_t* out_vtx_bits, uint32_t* out_idx, void* stream) {
    if (n < 1) return RMX_EINVAL;
    const uint64_t quads = static_cast<uint64_t>(n) * n;
    if (quads * 5u >= (1ull << 32)) return RMX_ERANGE;
    if (!out_vtx_bits || !out_idx) return RMX_EINVAL;
    int grid = 0;
    int rc = grid_for_stream(quads * 10u, grid);
    if (rc) return rc;
    k_gen_grid_quads<<<grid, kBlock, 0, static_cast<cudaStream_t>(stream)>>>(n, quads, out_vtx_bits, out_idx);
    RMX_CHECK(cudaGetLastError());
    return RMX_OK;
}

}  // extern "C"
