// sketch.cu — K1: fused count-sketch / higher-order count-sketch projection,
// discretisation and table-key packing for sm_100a.
//
// What it computes (per point p, per bin l):
//   y_l = sum_{j: bin(j)=l} sign(j) p_j          CS: PAPER.md:205; HCS: PAPER.md:212-215
//   E2LSH family: z_l = floor((sqrt(m) y_l + b_l)/w)
//   SRP family:   bit_l = [y_l > 0]
//   key_t = pack/fingerprint of (z|bit)_{tK..tK+K-1}       PAPER.md:155 + DESIGN.md B1, B10
//
// Design (B200-first, HBM-bound): a CTA of 16 warps owns a tile of 32 points;
// lane == point.  The tile's coordinates are staged in shared memory TRANSPOSED
// (word (k>>2)*129 + (k&3)*32 + p) so that (a) the staging stores of coalesced
// 128-bit row loads and (b) the per-bin gathers "all 32 lanes read coordinate k
// of their own point" are both bank-conflict free.  While the warps gather the
// current chunk, the next chunk's 128-bit loads are already in flight in
// registers (register file = second stage buffer; 32 x 1024 fp32 = 128 KB per
// tile would not fit twice in shared memory).  Warps own whole tables, so the
// bins of a table are summed, discretised and folded into the key in registers
// and each key is written once, coalesced (32 x 8 B per warp store).
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.hpp"

namespace lshb {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ float4 ldg_stream_f4(const float* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ float ldg_stream_f1(const float* p) {
    float r;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
    return r;
}

__device__ __forceinline__ uint64_t fmix64_dev(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// floor(q) as int32 with sticky overflow flags (DESIGN.md §K1 discretisation).
// Fast path |q| < 2^22: q + 1.5*2^23 rounded toward -inf has floor(q) in its low
// mantissa bits (exact in fp32).
__device__ __forceinline__ int32_t floor_code(float q, int* flags) {
    if (fabsf(q) < 4194304.0f) {
        float r = __fadd_rd(q, 12582912.0f);
        return __float_as_int(r) - 0x4B400000;
    }
    if (q != q) {
        atomicOr(flags, 2);
        return 0;
    }
    float fq = floorf(q);
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

// Discretise one bin and fold it into the running table key (shared by every
// projection kernel so the arithmetic is identical across schemes).
struct KeyAcc {
    uint64_t f;
    __device__ __forceinline__ void init(int e2lsh) { f = e2lsh ? LSHB_FNV_OFFSET : 0ull; }
    __device__ __forceinline__ void add(float y, int l, int kk, int64_t row, bool valid, int m, const DiscretizeDev& dz,
                                        const HashOut& out) {
        if (dz.e2lsh) {
            float q = fmaf(y, dz.c_scale, __ldg(dz.c_off + l));
            int32_t z = floor_code(q, dz.flags);
            f = (f ^ (uint64_t)(uint32_t)z) * LSHB_FNV_PRIME;
            if (out.codes && valid) out.codes[row * m + l] = z;
        } else {
            uint64_t bit = y > 0.0f ? 1ull : 0ull;
            f |= bit << kk;
            if (out.bits && valid && bit) atomicOr(&out.bits[row * ((m + 31) >> 5) + (l >> 5)], 1u << (l & 31));
        }
        if (out.proj && valid) out.proj[row * m + l] = y;
    }
    __device__ __forceinline__ uint64_t key(int e2lsh) const { return e2lsh ? fmix64_dev(f) : f; }
};

template <int VPT, bool VEC>
__global__ void __launch_bounds__(kThreads, 1)
    sketch_kernel(SketchPlanDev plan, DiscretizeDev dz, const float* __restrict__ X, int64_t n, int64_t ld,
                  HashOut out) {
    extern __shared__ __align__(16) float smem[];
    constexpr int Q = 64 * VPT;
    constexpr int Q4 = Q / 4;                 // float4 per row of a chunk
    constexpr int RPI = kThreads / Q4;        // rows per load iteration (VEC path)
    float* T = smem;                          // [Q4][129] transposed tile
    float* ys = smem + Q4 * 129;              // [m][32] partial bins (multi-chunk only)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = (n + 31) >> 5;
    const int m = plan.m, K = plan.K, L = plan.L, d = plan.d, nch = plan.nchunks;
    int64_t tile = blockIdx.x;
    if (tile >= ntiles) return;

    float4 buf[VPT];

    auto load = [&](int64_t tl, int c) {
        const int k0 = c * Q;
        const int Qc = min(Q, d - k0);
        if constexpr (VEC) {
            const int r0 = tid / Q4, c4 = tid % Q4;
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                const int r = r0 + v * RPI;
                const int64_t row = tl * 32 + r;
                if (row < n && 4 * c4 < Qc) buf[v] = ldg_stream_f4(X + row * ld + k0 + 4 * c4);
                else buf[v] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        } else {
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                float e[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int f = tid + kThreads * (4 * v + q);
                    const int r = f / Q, k = f % Q;
                    const int64_t row = tl * 32 + r;
                    e[q] = (row < n && k < Qc) ? ldg_stream_f1(X + row * ld + k0 + k) : 0.f;
                }
                buf[v] = make_float4(e[0], e[1], e[2], e[3]);
            }
        }
    };
    auto store = [&]() {
        if constexpr (VEC) {
            const int r0 = tid / Q4, c4 = tid % Q4;
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                const int r = r0 + v * RPI;
                float* dst = T + c4 * 129 + r;
                dst[0] = buf[v].x;
                dst[32] = buf[v].y;
                dst[64] = buf[v].z;
                dst[96] = buf[v].w;
            }
        } else {
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                const float e[4] = {buf[v].x, buf[v].y, buf[v].z, buf[v].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int f = tid + kThreads * (4 * v + q);
                    const int r = f / Q, k = f % Q;
                    T[(k >> 2) * 129 + (k & 3) * 32 + r] = e[q];
                }
            }
        }
    };

    int c = 0;
    load(tile, 0);
    while (true) {
        __syncthreads();  // previous gathers finished with T
        store();
        __syncthreads();
        int64_t ntile = tile;
        int nc = c + 1;
        if (nc == nch) {
            nc = 0;
            ntile += gridDim.x;
        }
        const bool has_next = ntile < ntiles;
        if (has_next) load(ntile, nc);  // in flight during the gathers below

        const bool first = (c == 0), last = (c == nch - 1);
        const int32_t* bp = plan.bin_ptr + (int64_t)c * (m + 1);
        const int64_t row = tile * 32 + lane;
        const bool valid = row < n;
        for (int t = warp; t < L; t += kWarps) {
            KeyAcc ka;
            ka.init(dz.e2lsh);
            int e = __ldg(bp + t * K);
            for (int kk = 0; kk < K; ++kk) {
                const int l = t * K + kk;
                const int e1 = __ldg(bp + l + 1);
                float acc = first ? 0.0f : ys[l * 32 + lane];
                for (; e < e1; ++e) {
                    const uint32_t en = __ldg(plan.entries + e);
                    const uint32_t v = __float_as_uint(T[(en & 0x7fffffffu) + lane]) ^ (en & 0x80000000u);
                    acc += __uint_as_float(v);
                }
                if (!last) {
                    ys[l * 32 + lane] = acc;
                } else {
                    ka.add(acc, l, kk, row, valid, m, dz, out);
                }
            }
            if (last && valid && out.keys) out.keys[(int64_t)t * n + row] = ka.key(dz.e2lsh);
        }
        if (!has_next) break;
        tile = ntile;
        c = nc;
    }
}

size_t sketch_smem_bytes(int Q, int m, int nchunks) {
    size_t b = (size_t)(Q / 4) * 129 * sizeof(float);
    if (nchunks > 1) b += (size_t)m * 32 * sizeof(float);
    return b;
}

template <int VPT, bool VEC>
static cudaError_t launch_t(const SketchPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n, int64_t ld,
                            HashOut out, int num_sms, cudaStream_t s) {
    const size_t smem = sketch_smem_bytes(64 * VPT, plan.m, plan.nchunks);
    cudaError_t e = cudaFuncSetAttribute(sketch_kernel<VPT, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = (n + 31) / 32;
    const int grid = (int)(ntiles < num_sms ? ntiles : num_sms);
    sketch_kernel<VPT, VEC><<<grid, kThreads, smem, s>>>(plan, dz, X, n, ld, out);
    return cudaGetLastError();
}

cudaError_t launch_sketch(const SketchPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n, int64_t ld,
                          HashOut out, int num_sms, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const bool vec = (plan.d % 4 == 0) && (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
#define LSHB_CASE(V)                                                                   \
    case V:                                                                            \
        return vec ? launch_t<V, true>(plan, dz, X, n, ld, out, num_sms, s)           \
                   : launch_t<V, false>(plan, dz, X, n, ld, out, num_sms, s);
    switch (plan.vpt) {
        LSHB_CASE(1)
        LSHB_CASE(2)
        LSHB_CASE(4)
        LSHB_CASE(8)
        LSHB_CASE(16)
        default:
            return cudaErrorInvalidValue;
    }
#undef LSHB_CASE
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
    KeyAcc ka;
    ka.init(dz.e2lsh);
    HashOut o2 = out;
    o2.proj = nullptr;
    for (int kk = 0; kk < K; ++kk) {
        const int l = t * K + kk;
        const float y = valid ? Y[row * m + l] : 0.f;
        ka.add(y, l, kk, row, valid, m, dz, o2);
    }
    if (valid && out.keys) out.keys[(int64_t)t * n + row] = ka.key(dz.e2lsh);
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
