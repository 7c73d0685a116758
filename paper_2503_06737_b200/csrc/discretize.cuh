// discretize.cuh — the device arithmetic every projection kernel shares, so codes
// and keys are bit-identical whichever kernel produced the projection.
//   floor_code: z = floor(q) as int32 (reading B9, floor toward -inf) with sticky
//               overflow / NaN flags (LSH_EOVERFLOW, include/lsh.h).  Fast path
//               |q| < 2^22: q + 1.5*2^23 rounded toward -inf holds floor(q) in its
//               low mantissa bits (exact in fp32).
//   FpKey:      the E2LSH table key of reading B10: two 32-bit Horner
//               lanes over the K codes, u_k = z_k as a two's-complement word,
//               a <- a*FP_A + u_k, b <- b*FP_B + u_k from 0, key = fmix64(a:b).
//   fmix64:     SplitMix64 output finaliser.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lshb {

#define LSHB_FP_A 0x9E3779B1u
#define LSHB_FP_B 0x85EBCA77u
// fp32 bit pattern of q + 1.5*2^23 for |q| < 2^22 is 0x4B400000 + floor(q)
#define LSHB_FLOOR_BIAS 0x4B400000u

__host__ __device__ __forceinline__ uint64_t fmix64_dev(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// sum_{j<K} mult^j mod 2^32: a Horner lane fed u_k + c instead of u_k ends c * this
// higher, so a kernel can hash biased words and subtract once per table.
__host__ __device__ constexpr uint32_t fp_geom(uint32_t mult, int K) {
    uint32_t s = 0, p = 1;
    for (int j = 0; j < K; ++j) {
        s += p;
        p *= mult;
    }
    return s;
}

struct FpKey {
    uint32_t a = 0, b = 0;
    __device__ __forceinline__ void add(uint32_t u) {
        a = a * LSHB_FP_A + u;
        b = b * LSHB_FP_B + u;
    }
    // lanes fed (u_k + LSHB_FLOOR_BIAS) for K codes: remove the bias
    __device__ __forceinline__ void unbias(int K) {
        a -= LSHB_FLOOR_BIAS * fp_geom(LSHB_FP_A, K);
        b -= LSHB_FLOOR_BIAS * fp_geom(LSHB_FP_B, K);
    }
    __device__ __forceinline__ uint64_t key() const { return fmix64_dev(((uint64_t)a << 32) | b); }
};

__device__ __forceinline__ int32_t floor_code(float q, int* flags) {
    if (fabsf(q) < 4194304.0f) return __float_as_int(__fadd_rd(q, 12582912.0f)) - (int32_t)LSHB_FLOOR_BIAS;
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
