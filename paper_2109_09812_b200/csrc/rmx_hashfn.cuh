// rmx_hashfn.cuh -- the 32-bit key hash of hash mode (rmx_hash.cuh): murmur3-style mixing of
// the key words and the murmur3 finaliser.  tests/test_gpu_hash.py mirrors it in numpy.
#pragma once

#include <cstdint>

namespace rmx {

__device__ __forceinline__ uint32_t hash_word(uint32_t h, uint32_t k) {
    k *= 0xcc9e2d51u;
    k = (k << 15) | (k >> 17);
    k *= 0x1b873593u;
    h ^= k;
    h = (h << 13) | (h >> 19);
    return h * 5u + 0xe6546b64u;
}

__device__ __forceinline__ uint32_t hash_final(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    return h ^ (h >> 16);
}

template <int D_CT>
__device__ __forceinline__ uint32_t hash_key(const uint32_t* k, int D) {
    uint32_t h = 0x9747b28cu;
    if constexpr (D_CT > 0) {
#pragma unroll
        for (int c = 0; c < D_CT; ++c) h = hash_word(h, k[c]);
    } else {
        for (int c = 0; c < D; ++c) h = hash_word(h, k[c]);
    }
    return hash_final(h);
}

}  // namespace rmx
