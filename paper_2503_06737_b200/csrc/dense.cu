// dense.cu — the dense O(md) E2LSH / SRP projection the sketches replace
// (PAPER.md:169 eq:datar_lsh, :187 Def. SRP; Table 1).
//
// Y = X R^T with R the m x d Gaussian matrix drawn by the host and rounded to
// bf16 (reading B13, so that a tensor-core product with it is exact).
// This translation unit holds the CUDA-core reference implementation (fp32 FMA,
// exact bf16 -> fp32 widening of R); the discretisation runs in
// keys_from_proj_kernel (sketch.cu) with the same arithmetic as the sketches.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.hpp"

namespace lshb {

constexpr int BM = 64, BN = 64, BK = 32;

__global__ void __launch_bounds__(256) dense_gemm_f32_kernel(const float* __restrict__ X, int64_t n, int64_t ld,
                                                             const uint16_t* __restrict__ R, int m, int d,
                                                             float* __restrict__ Y) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t row0 = (int64_t)blockIdx.y * BM;
    const int col0 = blockIdx.x * BN;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < d; k0 += BK) {
        for (int i = threadIdx.x; i < BM * BK; i += 256) {
            const int r = i / BK, k = i % BK;
            const int64_t gr = row0 + r;
            As[k][r] = (gr < n && k0 + k < d) ? X[gr * ld + k0 + k] : 0.f;
            const int gc = col0 + r;
            float bv = 0.f;
            if (gc < m && k0 + k < d) {
                const uint32_t bits = (uint32_t)R[(int64_t)gc * d + k0 + k] << 16;
                bv = __uint_as_float(bits);
            }
            Bs[k][r] = bv;
        }
        __syncthreads();
#pragma unroll 8
        for (int k = 0; k < BK; ++k) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t gr = row0 + ty * 4 + i;
        if (gr >= n) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gc = col0 + tx * 4 + j;
            if (gc < m) Y[gr * m + gc] = acc[i][j];
        }
    }
}

cudaError_t launch_dense_gemm_f32(const float* X, int64_t n, int64_t ld, const uint16_t* R, int m, int d, float* Y,
                                  cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    dim3 grid((m + BN - 1) / BN, (unsigned)((n + BM - 1) / BM));
    dense_gemm_f32_kernel<<<grid, 256, 0, s>>>(X, n, ld, R, m, d, Y);
    return cudaGetLastError();
}

}  // namespace lshb
