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

#include "discretize.cuh"
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



// Discretise one bin and fold it into the running table key (shared by every
// projection kernel so the arithmetic is identical across schemes).
template <bool E2>
struct KeyAccT {
    uint64_t f;
    __device__ __forceinline__ KeyAccT() : f(E2 ? LSHB_FNV_OFFSET : 0ull) {}
    // q-path for E2LSH: z = floor(y * c_scale + c_off_l) (= floor((sqrt(m) y + b)/w) for
    // power-of-two w, a single fp32 rounding); SRP: bit = [y > 0].
    __device__ __forceinline__ int32_t add(float y, float coff, int kk, int* flags) {
        if constexpr (E2) {
            (void)kk;
            const int32_t z = floor_code(y, flags);
            f = (f ^ (uint64_t)(uint32_t)z) * LSHB_FNV_PRIME;
            return z;
        } else {
            (void)coff;
            (void)flags;
            f |= (y > 0.0f ? 1ull : 0ull) << kk;
            return y > 0.0f ? 1 : 0;
        }
    }
    __device__ __forceinline__ uint64_t key() const { return E2 ? fmix64_dev(f) : f; }
};

// Legacy helper kept for keys_from_proj (runtime scheme flag).
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

// Shared-memory layout of the kernel (plan tables are loaded once per persistent CTA):
//   T    [(Q/4)*129 + 64] fp32  staged tile of 32 points, TRANSPOSED and sign-applied:
//                               coordinate k of point r at word (k>>2)*129 + (k&3)*32 + r.
//                               Both the staging stores (lanes = consecutive float4
//                               columns) and the gathers (lanes = points) are bank-
//                               conflict free.  Words ZW = (Q/4)*129 .. +31 stay 0.
//   bp   [m+1] u32              first bin-sorted index of every bin
//   cnt  [m]   u8               coordinates per bin (saturated at 255)
//   ent  [d]   u16              T word offset of the coordinate at each bin-sorted index
//   coff [m]   fp32             b_l / w
//   sgn  [ceil(d/32)] u32       bit j set: sign(j) = -1
//   pairs[2m]  u32              byte offsets of each bin's first two coordinates (zero slot if missing)
//   big  [L]   u32              bit k: bin k of table t has more than two coordinates
struct SketchSmem {
    size_t t, bp, cnt, ent, coff, sgn, pairs, big, total;
};
__host__ __device__ inline SketchSmem sketch_smem_layout(int Q, int m, int d, int L) {
    SketchSmem o{};
    size_t x = 0;
    o.t = x;
    x += ((size_t)(Q / 4) * 129 + 64) * 4;
    x = (x + 15) / 16 * 16;
    o.pairs = x;
    x += (size_t)m * 8;
    x = (x + 15) / 16 * 16;
    o.coff = x;
    x += (size_t)m * 4;
    x = (x + 15) / 16 * 16;
    o.bp = x;
    x += (size_t)(m + 1) * 4;
    x = (x + 15) / 16 * 16;
    o.cnt = x;
    x += ((size_t)m + 15) / 16 * 16;
    o.ent = x;
    x += ((size_t)d * 2 + 15) / 16 * 16;
    o.sgn = x;
    x += (size_t)((d + 31) / 32) * 4;
    o.big = x;
    x += (size_t)L * 4;
    o.total = (x + 15) / 16 * 16;
    return o;
}

// max.NaN: propagates NaN so one instruction checks both range and NaN/Inf.
__device__ __forceinline__ float fmax_nan_abs(float a, float q) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(fabsf(q)));
    return r;
}

template <int VPT, bool VEC, int KT, bool E2>
__global__ void __launch_bounds__(kThreads, 1)
    sketch_kernel(SketchPlanDev plan, DiscretizeDev dz, const float* __restrict__ X, int64_t n, int64_t ld,
                  HashOut out, int dbg) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int Q = 64 * VPT;
    constexpr int Q4 = Q / 4;                 // float4 per row of the tile
    constexpr int RPI = kThreads / Q4;        // rows per load iteration (VEC path)
    constexpr uint32_t ZW = (uint32_t)Q4 * 129u;
    const int m = plan.m, L = plan.L, d = plan.d;
    const int K = KT > 0 ? KT : plan.K;
    const SketchSmem so = sketch_smem_layout(Q, m, d, L);
    float* T = reinterpret_cast<float*>(smem_raw + so.t);
    uint32_t* s_bp = reinterpret_cast<uint32_t*>(smem_raw + so.bp);
    uint8_t* s_cnt = reinterpret_cast<uint8_t*>(smem_raw + so.cnt);
    uint16_t* s_ent = reinterpret_cast<uint16_t*>(smem_raw + so.ent);
    float* s_coff = reinterpret_cast<float*>(smem_raw + so.coff);
    uint32_t* s_sgn = reinterpret_cast<uint32_t*>(smem_raw + so.sgn);
    uint32_t* s_pairs = reinterpret_cast<uint32_t*>(smem_raw + so.pairs);
    uint32_t* s_big = reinterpret_cast<uint32_t*>(smem_raw + so.big);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = (n + 31) >> 5;
    int64_t tile = blockIdx.x;
    if (tile >= ntiles) return;

    for (int i = tid; i <= m; i += kThreads) s_bp[i] = __ldg(plan.bin_ptr + i);
    for (int i = tid; i < m; i += kThreads) {
        const uint32_t cn = __ldg(plan.bin_ptr + i + 1) - __ldg(plan.bin_ptr + i);
        s_cnt[i] = (uint8_t)(cn < 255u ? cn : 255u);
        s_coff[i] = E2 ? __ldg(dz.c_off + i) : 0.f;
        s_pairs[2 * i] = __ldg(plan.pairs + 2 * i);
        s_pairs[2 * i + 1] = __ldg(plan.pairs + 2 * i + 1);
    }
    for (int i = tid; i < d; i += kThreads) s_ent[i] = __ldg(plan.pos + i);
    for (int i = tid; i < (d + 31) / 32; i += kThreads) s_sgn[i] = __ldg(plan.sign_bits + i);
    for (int i = tid; i < L; i += kThreads) s_big[i] = __ldg(plan.bigmask + i);
    for (int i = tid; i < 64; i += kThreads) T[ZW + i] = 0.f;
    __syncthreads();

    float4 buf[VPT];
    // this thread's 4 staging columns (VEC path): sign masks, fixed for the kernel
    const int c4 = tid % Q4, r0 = tid / Q4;
    const bool col_ok = 4 * c4 < d;
    uint32_t sm0 = 0, sm1 = 0, sm2 = 0, sm3 = 0;
    if (VEC && col_ok) {
        const int k = 4 * c4;
        const uint32_t w = s_sgn[k >> 5] >> (k & 31);  // 4 | k: never straddles a word
        sm0 = (w & 1u) << 31;
        sm1 = ((w >> 1) & 1u) << 31;
        sm2 = ((w >> 2) & 1u) << 31;
        sm3 = ((w >> 3) & 1u) << 31;
    }

    auto load = [&](int64_t tl) {
        if constexpr (VEC) {
            if (col_ok) {
                const float* src = X + (tl * 32 + r0) * ld + 4 * c4;
                const int64_t stride = (int64_t)RPI * ld;
                if (tl * 32 + 32 <= n) {  // full tile: no row predicates
#pragma unroll
                    for (int v = 0; v < VPT; ++v) buf[v] = ldg_stream_f4(src + v * stride);
                } else {
                    const int64_t rows_left = n - tl * 32 - r0;
#pragma unroll
                    for (int v = 0; v < VPT; ++v)
                        buf[v] = v * RPI < rows_left ? ldg_stream_f4(src + v * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
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
                    e[q] = (row < n && k < d) ? ldg_stream_f1(X + row * ld + k) : 0.f;
                }
                buf[v] = make_float4(e[0], e[1], e[2], e[3]);
            }
        }
    };
    auto store = [&]() {
        if constexpr (VEC) {
            if (col_ok) {
                float* dst = T + c4 * 129 + r0;
#pragma unroll
                for (int v = 0; v < VPT; ++v) {
                    dst[v * RPI] = __uint_as_float(__float_as_uint(buf[v].x) ^ sm0);
                    dst[v * RPI + 32] = __uint_as_float(__float_as_uint(buf[v].y) ^ sm1);
                    dst[v * RPI + 64] = __uint_as_float(__float_as_uint(buf[v].z) ^ sm2);
                    dst[v * RPI + 96] = __uint_as_float(__float_as_uint(buf[v].w) ^ sm3);
                }
            }
        } else {
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                const float e[4] = {buf[v].x, buf[v].y, buf[v].z, buf[v].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int f = tid + kThreads * (4 * v + q);
                    const int r = f / Q, k = f % Q;
                    if (k < d) {
                        const uint32_t sg = ((s_sgn[k >> 5] >> (k & 31)) & 1u) << 31;
                        T[(k >> 2) * 129 + (k & 3) * 32 + r] = __uint_as_float(__float_as_uint(e[q]) ^ sg);
                    }
                }
            }
        }
    };

    load(tile);
    const float cs = dz.c_scale;
    const float* Tl = T + lane;
    while (true) {
        __syncthreads();  // previous gathers finished with T
        store();
        __syncthreads();
        const int64_t ntile = tile + gridDim.x;
        const bool has_next = ntile < ntiles;
        if (has_next) load(ntile);  // in flight during the gathers below
        const int64_t row = tile * 32 + lane;
        const bool valid = row < n;
        if constexpr (KT > 0) {
            // hot path: each bin's first two coordinates through `pairs` (branch-free; a
            // missing one reads the zero slot), rare fix-ups for fuller bins, then
            // discretise + key for the K bins of the table.  Two tables per iteration: their
            // fingerprint chains (16 dependent multiply steps each) interleave.
#pragma unroll 2
            for (int t = warp; t < L; t += kWarps) {
                float acc[KT];
                {
                    // two byte offsets per bin, read 2 bins per 128-bit load; one add each
                    const uint4* pp4 = reinterpret_cast<const uint4*>(s_pairs + t * KT * 2);
                    const char* Tb = reinterpret_cast<const char*>(Tl);
#pragma unroll
                    for (int i = 0; i < KT / 2; ++i) {
                        const uint4 v = pp4[i];
                        acc[2 * i] = *reinterpret_cast<const float*>(Tb + v.x) + *reinterpret_cast<const float*>(Tb + v.y);
                        acc[2 * i + 1] =
                            *reinterpret_cast<const float*>(Tb + v.z) + *reinterpret_cast<const float*>(Tb + v.w);
                    }
                }
                const uint32_t big = s_big[t];
                if (big) {
#pragma unroll
                    for (int kk = 0; kk < KT; ++kk) {
                        if ((big >> kk) & 1u) {
                            const int l = t * KT + kk;
                            for (uint32_t j = s_bp[l] + 2; j < s_bp[l + 1]; ++j) acc[kk] += Tl[s_ent[j]];
                        }
                    }
                }
                uint64_t f;
                if constexpr (E2) {
                    f = LSHB_FNV_OFFSET;
                    float qmax = 0.f;
                    const float4* co = reinterpret_cast<const float4*>(s_coff + t * KT);
#pragma unroll
                    for (int k4 = 0; k4 < KT / 4; ++k4) {
                        const float4 c4v = co[k4];
                        const float cc[4] = {c4v.x, c4v.y, c4v.z, c4v.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float q = fmaf(acc[4 * k4 + j], cs, cc[j]);
                            qmax = fmax_nan_abs(qmax, q);
                            const int32_t z = __float_as_int(__fadd_rd(q, 12582912.0f)) - 0x4B400000;
                            f = (f ^ (uint64_t)(uint32_t)z) * LSHB_FNV_PRIME;
                        }
                    }
                    if (!(qmax < 4194304.0f)) {
                        // rare: a code outside the fast floor range (or NaN/Inf): redo exactly
                        f = LSHB_FNV_OFFSET;
#pragma unroll
                        for (int kk = 0; kk < KT; ++kk) {
                            const int32_t z = floor_code(fmaf(acc[kk], cs, s_coff[t * KT + kk]), dz.flags);
                            f = (f ^ (uint64_t)(uint32_t)z) * LSHB_FNV_PRIME;
                        }
                    }
                    f = fmix64_dev(f);
                } else {
                    uint32_t sb = 0;
#pragma unroll
                    for (int kk = 0; kk < KT; ++kk) sb |= (acc[kk] > 0.0f ? 1u : 0u) << kk;
                    f = sb;
                }
                if (valid && out.keys) out.keys[(int64_t)t * n + row] = f;
            }
        } else {
            // generic K (and the debug outputs): sequential sum over each bin's coordinates
            for (int t = warp; t < L; t += kWarps) {
                uint64_t f = E2 ? LSHB_FNV_OFFSET : 0ull;
                for (int kk = 0; kk < K; ++kk) {
                    const int l = t * K + kk;
                    float acc = 0.0f;
                    for (uint32_t j = s_bp[l]; j < s_bp[l + 1]; ++j) acc += Tl[s_ent[j]];
                    int32_t z;
                    if constexpr (E2) {
                        z = floor_code(fmaf(acc, cs, s_coff[l]), dz.flags);
                        f = (f ^ (uint64_t)(uint32_t)z) * LSHB_FNV_PRIME;
                    } else {
                        z = acc > 0.0f ? 1 : 0;
                        f |= (uint64_t)z << kk;
                    }
                    if (dbg && valid) {
                        if (out.proj) out.proj[row * m + l] = acc;
                        if (E2 && out.codes) out.codes[row * m + l] = z;
                        if (!E2 && out.bits && z) atomicOr(&out.bits[row * ((m + 31) >> 5) + (l >> 5)], 1u << (l & 31));
                    }
                }
                if (valid && out.keys) out.keys[(int64_t)t * n + row] = E2 ? fmix64_dev(f) : f;
            }
        }
        if (!has_next) break;
        tile = ntile;
    }
}

size_t sketch_smem_bytes(int Q, int m, int d, int L) { return sketch_smem_layout(Q, m, d, L).total; }

template <int VPT, bool VEC, int KT, bool E2>
static cudaError_t launch_t(const SketchPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n, int64_t ld,
                            HashOut out, int num_sms, cudaStream_t s) {
    const size_t smem = sketch_smem_bytes(64 * VPT, plan.m, plan.d, plan.L);
    auto kern = sketch_kernel<VPT, VEC, KT, E2>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = (n + 31) / 32;
    const int grid = (int)(ntiles < num_sms ? ntiles : num_sms);
    const int dbg = (out.codes || out.bits || out.proj) ? 1 : 0;
    kern<<<grid, kThreads, smem, s>>>(plan, dz, X, n, ld, out, dbg);
    return cudaGetLastError();
}

template <int VPT, bool VEC>
static cudaError_t launch_k(const SketchPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n, int64_t ld,
                            HashOut out, int num_sms, cudaStream_t s) {
    const bool e2 = dz.e2lsh != 0;
    const bool dbg = out.codes || out.bits || out.proj;  // debug outputs: generic instantiation
    if (plan.K == 16 && !dbg)
        return e2 ? launch_t<VPT, VEC, 16, true>(plan, dz, X, n, ld, out, num_sms, s)
                  : launch_t<VPT, VEC, 16, false>(plan, dz, X, n, ld, out, num_sms, s);
    if (plan.K == 8 && !dbg)
        return e2 ? launch_t<VPT, VEC, 8, true>(plan, dz, X, n, ld, out, num_sms, s)
                  : launch_t<VPT, VEC, 8, false>(plan, dz, X, n, ld, out, num_sms, s);
    return e2 ? launch_t<VPT, VEC, 0, true>(plan, dz, X, n, ld, out, num_sms, s)
              : launch_t<VPT, VEC, 0, false>(plan, dz, X, n, ld, out, num_sms, s);
}

cudaError_t launch_sketch(const SketchPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n, int64_t ld,
                          HashOut out, int num_sms, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const bool vec = (plan.d % 4 == 0) && (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
    switch (plan.vpt) {
        case 1:
            return vec ? launch_k<1, true>(plan, dz, X, n, ld, out, num_sms, s)
                       : launch_k<1, false>(plan, dz, X, n, ld, out, num_sms, s);
        case 4:
            return vec ? launch_k<4, true>(plan, dz, X, n, ld, out, num_sms, s)
                       : launch_k<4, false>(plan, dz, X, n, ld, out, num_sms, s);
        case 16:
            return vec ? launch_k<16, true>(plan, dz, X, n, ld, out, num_sms, s)
                       : launch_k<16, false>(plan, dz, X, n, ld, out, num_sms, s);
        default:
            return cudaErrorInvalidValue;
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
