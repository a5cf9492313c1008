// rmx_hashfn.cuh -- the 32-bit key hash of hash mode (rmx_hash.cuh): per key word one
// xor-multiply step (a bijection of the running state), then an xor-shift-multiply finaliser
// that spreads every input bit into the top bits the hashed passes sort by.  Cheap on purpose
// (~11 instructions for D = 3): the hashed passes evaluate it twice per row and pass, and
// exactness never depends on its quality (only the bucket sizes do).  tests/test_gpu_hash.py
// mirrors it in numpy.
#pragma once

#include <cstdint>

namespace rmx {

template <int D_CT>
__device__ __forceinline__ uint32_t hash_key(const uint32_t* k, int D) {
    uint32_t h = 0x9747b28cu;
    if constexpr (D_CT > 0) {
#pragma unroll
        for (int c = 0; c < D_CT; ++c) h = (h ^ k[c]) * 0x9e3779b1u;
    } else {
        for (int c = 0; c < D; ++c) h = (h ^ k[c]) * 0x9e3779b1u;
    }
    h ^= h >> 15;
    h *= 0x85ebca77u;
    return h ^ (h >> 13);
}

// dedup table slot of a row: the top bits of a second multiply (the hash's own top bits are the
// row's bucket, shared by every row of a bucket)
__device__ __forceinline__ uint32_t hash_slot(uint32_t h, int bits) { return (h * 0x2545f491u) >> (32 - bits); }

}  // namespace rmx
