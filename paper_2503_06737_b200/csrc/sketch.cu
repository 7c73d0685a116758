// sketch.cu — K1 dispatch: picks the sketch_kernel instantiation
// (sketch_kernel.cuh) for a plan and a call; the K = 8 / 16 keys-only hot paths
// are instantiated in sketch_fast.cu.  Also the discretise + keys kernel for a
// materialised projection (dense debug outputs).
#include <cuda_runtime.h>
#include <stdint.h>

#include "sketch_kernel.cuh"

namespace lshb {

size_t sketch_smem_bytes(int Q, int m, int d, int L) { return sk::sketch_smem_layout(Q, m, d, L).total; }

template <int Q4>
static cudaError_t launch_q(const SketchPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n, int64_t ld,
                            HashOut out, int num_sms, cudaStream_t s, bool vec) {
    const bool e2 = dz.e2lsh != 0;
    const bool dbg = out.codes || out.bits || out.proj;  // debug outputs: generic instantiation
    if (vec && !dbg && (plan.K == 16 || plan.K == 8)) return launch_sketch_fast(plan, dz, X, n, ld, out, num_sms, s);
    if (vec)
        return e2 ? sk::launch_t<Q4, true, 0, true>(plan, dz, X, n, ld, out, num_sms, s)
                  : sk::launch_t<Q4, true, 0, false>(plan, dz, X, n, ld, out, num_sms, s);
    return e2 ? sk::launch_t<Q4, false, 0, true>(plan, dz, X, n, ld, out, num_sms, s)
              : sk::launch_t<Q4, false, 0, false>(plan, dz, X, n, ld, out, num_sms, s);
}

static bool sketch_vec_ok(const SketchPlanDev& plan, const float* X, int64_t ld) {
    return (plan.d % 4 == 0) && (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
}

cudaError_t launch_sketch(const SketchPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n, int64_t ld,
                          HashOut out, int num_sms, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const bool vec = sketch_vec_ok(plan, X, ld);
    switch (plan.vpt) {
        case 1: return launch_q<16>(plan, dz, X, n, ld, out, num_sms, s, vec);
        case 4: return launch_q<64>(plan, dz, X, n, ld, out, num_sms, s, vec);
        case 16: return launch_q<256>(plan, dz, X, n, ld, out, num_sms, s, vec);
        default: return cudaErrorInvalidValue;
    }
}

// ---------------------------------------------------------------------------
// Discretise + keys from a materialised projection Y [n][m] (dense baseline path
// until the fused tcgen05 epilogue takes over; also a generic fallback).
// ---------------------------------------------------------------------------
__global__ void keys_from_proj_kernel(const float* __restrict__ Y, int64_t n, int m, int L, int K, DiscretizeDev dz,
                                      HashOut out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp_global = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t ntiles = (n + 31) >> 5;
    const int64_t tile = warp_global / L;
    const int t = (int)(warp_global % L);
    if (tile >= ntiles) return;
    const int64_t row = tile * 32 + lane;
    const bool valid = row < n;
    FpKey fk;
    uint64_t sbits = 0;
    for (int kk = 0; kk < K; ++kk) {
        const int l = t * K + kk;
        const float y = valid ? Y[row * m + l] : 0.f;
        if (dz.e2lsh) {
            const int32_t z = floor_code(fmaf(y, dz.c_scale, __ldg(dz.c_off + l)), dz.flags);
            fk.add((uint32_t)z);
            if (out.codes && valid) out.codes[row * m + l] = z;
        } else {
            const uint64_t bit = y > 0.0f ? 1ull : 0ull;
            sbits |= bit << kk;
            if (out.bits && valid && bit) atomicOr(&out.bits[row * ((m + 31) >> 5) + (l >> 5)], 1u << (l & 31));
        }
    }
    if (valid && out.keys) out.keys[(int64_t)t * n + row] = dz.e2lsh ? fk.key() : sbits;
}

cudaError_t launch_keys_from_proj(const float* Y, int64_t n, int m, int L, int K, const DiscretizeDev& dz,
                                  HashOut out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int64_t warps = ((n + 31) / 32) * L;
    const int64_t blocks = (warps * 32 + 255) / 256;
    keys_from_proj_kernel<<<(unsigned)blocks, 256, 0, s>>>(Y, n, m, L, K, dz, out);
    return cudaGetLastError();
}

}  // namespace lshb
