// DSMEM scatter microbenchmark for the map fill (K3b): pairs (org, new_idx)
// whose org is random within a window owned by a thread-block cluster; every
// CTA of the cluster reads a slice of the window's pairs and stores new_idx
// into the shared memory of the CTA that owns org (st.shared::cluster), then
// every CTA writes its window slice out coalesced.  Compared with the direct
// global scatter map[org] = new_idx (L2-merged partial sectors).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_fill dsmem_fill.cu
//   ./dsmem_fill [n_rows=157500000]
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <numeric>
#include <random>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("%s: %s\n", #x, cudaGetErrorString(e)); std::exit(1); } } while (0)

constexpr int kThreads = 1024;

// pairs are bucket-major: bucket b holds every org in [b*W, (b+1)*W), random order
template <int CL, int SLICE_LOG2>
__global__ void __launch_bounds__(kThreads, 1) k_fill_dsmem(const uint2* pairs, uint32_t n, uint32_t* map) {
    extern __shared__ __align__(16) uint32_t s_win[];
    cg::cluster_group cl = cg::this_cluster();
    constexpr uint32_t kSlice = 1u << SLICE_LOG2;
    constexpr uint32_t kWin = kSlice * CL;
    const uint32_t rank = cl.block_rank();
    const uint32_t bucket = blockIdx.x / CL;
    const uint64_t b0 = static_cast<uint64_t>(bucket) * kWin;
    const uint32_t nb = static_cast<uint32_t>(n - b0 < kWin ? n - b0 : kWin);
    cl.sync();  // every CTA of the cluster is running before remote stores
    const uint2* src = pairs + b0;
    for (uint32_t i = rank * kThreads + threadIdx.x; i < nb; i += CL * kThreads) {
        const uint2 p = __ldcs(src + i);
        const uint32_t off = p.x - static_cast<uint32_t>(b0);
        uint32_t* dst = cl.map_shared_rank(s_win, off >> SLICE_LOG2);
        dst[off & (kSlice - 1)] = p.y;
    }
    cl.sync();
    const uint64_t base = b0 + static_cast<uint64_t>(rank) * kSlice;
    if (base < n) {
        const uint32_t m = static_cast<uint32_t>(n - base < kSlice ? n - base : kSlice);
        for (uint32_t j = threadIdx.x; j < m; j += kThreads) __stcs(map + base + j, s_win[j]);
    }
}

__global__ void k_fill_direct(const uint2* pairs, uint32_t n, uint32_t* map) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) {
        const uint2 p = __ldcs(pairs + i);
        map[p.x] = p.y;
    }
}

template <int CL, int SLICE_LOG2>
float run_dsmem(const uint2* d_pairs, uint32_t n, uint32_t* d_map) {
    auto kern = k_fill_dsmem<CL, SLICE_LOG2>;
    const size_t smem = (size_t{1} << SLICE_LOG2) * 4;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    if (CL > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const uint32_t win = (1u << SLICE_LOG2) * CL;
    const uint32_t buckets = (n + win - 1) / win;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(buckets * CL);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int w = 0; w < 2; ++w) CK(cudaLaunchKernelEx(&cfg, kern, d_pairs, n, d_map));
    CK(cudaEventRecord(a));
    const int reps = 5;
    for (int r = 0; r < reps; ++r) CK(cudaLaunchKernelEx(&cfg, kern, d_pairs, n, d_map));
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms / reps;
}

int main(int argc, char** argv) {
    const uint32_t n = argc > 1 ? static_cast<uint32_t>(std::atoll(argv[1])) : 157500000u;
    // bucket-major pairs: within each 2^18-row bucket a random permutation (the widest window tested)
    std::vector<uint2> h(n);
    std::mt19937 rng(1);
    const uint32_t W = 1u << 18;
    std::vector<uint32_t> perm;
    for (uint64_t b0 = 0; b0 < n; b0 += W) {
        const uint32_t m = static_cast<uint32_t>(std::min<uint64_t>(W, n - b0));
        perm.resize(m);
        std::iota(perm.begin(), perm.end(), 0u);
        std::shuffle(perm.begin(), perm.end(), rng);
        for (uint32_t i = 0; i < m; ++i) h[b0 + i] = make_uint2(static_cast<uint32_t>(b0) + perm[i], perm[i] ^ 0x5a5a5u);
    }
    uint2* d_pairs;
    uint32_t *d_map, *d_ref;
    CK(cudaMalloc(&d_pairs, sizeof(uint2) * n));
    CK(cudaMalloc(&d_map, 4ull * n));
    CK(cudaMalloc(&d_ref, 4ull * n));
    CK(cudaMemcpy(d_pairs, h.data(), sizeof(uint2) * n, cudaMemcpyHostToDevice));
    // direct scatter
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    k_fill_direct<<<(n + 255) / 256, 256>>>(d_pairs, n, d_ref);
    CK(cudaEventRecord(a));
    for (int r = 0; r < 5; ++r) k_fill_direct<<<(n + 255) / 256, 256>>>(d_pairs, n, d_ref);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    std::printf("direct scatter (2^18-row windows): %.3f ms\n", ms / 5);
    auto check = [&](const char* name, float t) {
        std::vector<uint32_t> x(n), y(n);
        CK(cudaMemcpy(x.data(), d_map, 4ull * n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(y.data(), d_ref, 4ull * n, cudaMemcpyDeviceToHost));
        std::printf("%s: %.3f ms  %s\n", name, t, x == y ? "ok" : "MISMATCH");
        CK(cudaMemset(d_map, 0, 4ull * n));
    };
    check("dsmem cluster 8 x 32K rows (2^18 window)", run_dsmem<8, 15>(d_pairs, n, d_map));
    check("dsmem cluster 16 x 16K rows (2^18 window)", run_dsmem<16, 14>(d_pairs, n, d_map));
    return 0;
}
