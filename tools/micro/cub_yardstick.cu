// Yardstick only (never on the product path): CUB DeviceRadixSort::SortPairs on
// the shape of one C2 packed sort -- 157.5M (u32 key, u32 origin) pairs -- so the
// per-pass time of the hand-written LSD passes can be compared with the
// library's onesweep on the same box.  Also a plain device copy of the same
// bytes for the HBM ceiling.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cub_yardstick tools/micro/cub_yardstick.cu
#include <cstdio>
#include <cstdint>
#include <cub/cub.cuh>

__global__ void fill(uint32_t* k, uint32_t* v, uint32_t n, uint32_t mask) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t x = i * 2654435761u;
        x ^= x >> 15;
        x *= 0x2c1b3c6du;
        x ^= x >> 12;
        k[i] = x & mask;
        v[i] = i;
    }
}

__global__ void copy4(const uint4* a, uint4* b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = __ldcs(a + i);
}

int main(int argc, char** argv) {
    const uint32_t n = argc > 1 ? (uint32_t)atoll(argv[1]) : 157500000u;
    uint32_t *k0, *k1, *v0, *v1;
    cudaMalloc(&k0, n * 4ull);
    cudaMalloc(&k1, n * 4ull);
    cudaMalloc(&v0, n * 4ull);
    cudaMalloc(&v1, n * 4ull);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int bits_list[] = {32, 24, 16, 8};
    for (int bits : bits_list) {
        const uint32_t mask = bits == 32 ? 0xFFFFFFFFu : ((1u << bits) - 1u);
        size_t tmp = 0;
        cub::DoubleBuffer<uint32_t> kb(k0, k1), vb(v0, v1);
        cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, n, 0, bits);
        void* t = nullptr;
        cudaMalloc(&t, tmp);
        float best = 1e9f;
        for (int rep = 0; rep < 6; ++rep) {
            fill<<<1184, 256>>>(k0, v0, n, mask);
            cub::DoubleBuffer<uint32_t> kb2(k0, k1), vb2(v0, v1);
            cudaEventRecord(a);
            cub::DeviceRadixSort::SortPairs(t, tmp, kb2, vb2, n, 0, bits);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) best = ms < best ? ms : best;
        }
        const int passes = (bits + 7) / 8;
        printf("{\"what\": \"cub SortPairs u32/u32\", \"n\": %u, \"bits\": %d, \"ms\": %.4f, \"ms_per_8bit_pass\": %.4f, "
               "\"gbs_per_pass_16B_rows\": %.1f}\n",
               n, bits, best, best / passes, 16.0 * n / (best / passes * 1e-3) / 1e9);
        cudaFree(t);
    }
    // keys only, 32 bits
    {
        size_t tmp = 0;
        cub::DoubleBuffer<uint32_t> kb(k0, k1);
        cub::DeviceRadixSort::SortKeys(nullptr, tmp, kb, n, 0, 32);
        void* t = nullptr;
        cudaMalloc(&t, tmp);
        float best = 1e9f;
        for (int rep = 0; rep < 6; ++rep) {
            fill<<<1184, 256>>>(k0, v0, n, 0xFFFFFFFFu);
            cub::DoubleBuffer<uint32_t> kb2(k0, k1);
            cudaEventRecord(a);
            cub::DeviceRadixSort::SortKeys(t, tmp, kb2, n, 0, 32);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) best = ms < best ? ms : best;
        }
        printf("{\"what\": \"cub SortKeys u32\", \"n\": %u, \"bits\": 32, \"ms\": %.4f}\n", n, best);
        cudaFree(t);
    }
    // plain copy of 8 B x n (read + write 16 B per row)
    {
        const size_t n16 = n * 8ull / 16;
        float best = 1e9f;
        for (int rep = 0; rep < 6; ++rep) {
            cudaEventRecord(a);
            copy4<<<148 * 8, 512>>>(reinterpret_cast<const uint4*>(k0), reinterpret_cast<uint4*>(k1), n16 / 2);
            copy4<<<148 * 8, 512>>>(reinterpret_cast<const uint4*>(v0), reinterpret_cast<uint4*>(v1), n16 / 2);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) best = ms < best ? ms : best;
        }
        printf("{\"what\": \"copy 8 B per row\", \"n\": %u, \"ms\": %.4f, \"gbs\": %.1f}\n", n, best,
               16.0 * n / (best * 1e-3) / 1e9);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
