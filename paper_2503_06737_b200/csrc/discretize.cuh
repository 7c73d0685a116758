// discretize.cuh — the device arithmetic every projection kernel shares, so codes
// and keys are bit-identical whichever kernel produced the projection.
//   floor_code: z = floor(q) as int32 (reading B9, floor toward -inf) with sticky
//               overflow / NaN flags (LSH_EOVERFLOW, include/lsh.h).  Fast path
//               |q| < 2^22: q + 1.5*2^23 rounded toward -inf holds floor(q) in its
//               low mantissa bits (exact in fp32).
//   fmix64:     SplitMix64 output finaliser, the last step of the E2LSH table key
//               (reading B10: FNV-1a-64 over the K codes, then fmix64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lshb {

__device__ __forceinline__ uint64_t fmix64_dev(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ int32_t floor_code(float q, int* flags) {
    if (fabsf(q) < 4194304.0f) return __float_as_int(__fadd_rd(q, 12582912.0f)) - 0x4B400000;
    if (q != q) {
        atomicOr(flags, 2);
        return 0;
    }
    const float fq = floorf(q);
    if (fq >= 2147483648.0f) {
        atomicOr(flags, 1);
        return INT32_MAX;
    }
    if (fq < -2147483648.0f) {
        atomicOr(flags, 1);
        return INT32_MIN;
    }
    return (int32_t)fq;
}

}  // namespace lshb
