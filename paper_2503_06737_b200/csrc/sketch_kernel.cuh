// sketch_kernel.cuh — K1: fused count-sketch projection, discretisation and
// table-key packing for sm_100a.  Included by sketch.cu (generic
// instantiations + dispatch) and sketch_fast.cu (the K = 8 / 16 keys-only paths),
// so the two translation units compile in parallel.
//
// What it computes (per point p, per bin l):
//   y_l = sum_{j: h(j)=l} s(j) p_j                          CS: PAPER.md:205 (eq:eq_cs)
//   E2LSH family: z_l = floor((sqrt(m) y_l + b_l)/w)        PAPER.md:314 (Def. CS-E2LSH)
//   SRP family:   bit_l = [y_l > 0]                         PAPER.md:918-920 (Def. CS-SRP)
//   key_t = SRP bits packed / E2LSH fingerprint of z_{tK..tK+K-1}   PAPER.md:155 + B1, B10
//
// Design (B200-first, HBM-bound): persistent CTAs of 16 warps, one per SM; a CTA
// owns a tile of 32 points, lane == point.  The tile's coordinates are staged in
// shared memory TRANSPOSED and sign-applied: coordinate k of point r at word
// (k>>2)*kSketchColWords + (k&3)*32 + r.  Each thread loads a 4 x 4 block (4
// consecutive rows of one float4 column, coalesced 128-bit loads: a warp reads 512
// contiguous bytes of a row) and writes it back transposed as four 128-bit shared
// stores, one per coordinate (the 132-word column pitch keeps the 8 lanes of each
// store phase on distinct bank groups).  The gathers "all 32 lanes read coordinate
// k of their own point" are conflict-free.  While the warps gather the current
// tile, the next tile's loads are in flight in registers (32 x 1024 fp32 = 128 KB
// per tile would not fit twice in shared memory).  Warps own whole tables: a
// table's K bins are summed, discretised and folded into its key in registers,
// and each key is written once, coalesced (32 x 8 B per warp store).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "discretize.cuh"
#include "internal.hpp"

#ifndef LSHB_SK_QUAD
// keys-only path with four tables per warp and 128-bit gathers of four points:
// 1 = E2LSH keys only, 2 = E2LSH and SRP (default), 0 = never (lane per point)
#define LSHB_SK_QUAD 2
#endif
#ifndef LSHB_SK_QPRE
#define LSHB_SK_QPRE 0      // four-table path: pair-offset vectors read before the fold
#endif
#ifndef LSHB_SK_TUNROLL
#define LSHB_SK_TUNROLL 2   // tables per iteration of a warp's keys-only loop
#endif

namespace lshb {
namespace sk {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kTUnroll = LSHB_SK_TUNROLL;
constexpr int CW = kSketchColWords;   // words per staged float4 column (4 coordinates x 32 points + pad)

#ifndef LSHB_SK_LDHINT
// streamed X loads: 0 plain, 1 L2::256B prefetch size, 2 L2::evict_first policy, 3 both,
// 4 evict_first in the E2LSH instantiations only
#define LSHB_SK_LDHINT 0
#endif
#ifndef LSHB_SK_ST128
// four-table path, a lane's four keys: 0 four 64-bit stores, 1 two 128-bit stores, 2 one
// 256-bit store (3: with .cs) when the address is aligned, else the narrower forms
#define LSHB_SK_ST128 2
#endif
#if LSHB_SK_LDHINT == 1 || LSHB_SK_LDHINT == 3
#define LSHB_SK_LDQ ".L2::256B"
#else
#define LSHB_SK_LDQ ""
#endif
template <bool EF>
__device__ __forceinline__ float4 ldg_stream_f4(const float* p) {
    float4 r;
    if constexpr (EF) {
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint" LSHB_SK_LDQ ".v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                     : "l"(p), "l"(pol));
    } else {
        asm volatile("ld.global.nc.L1::no_allocate" LSHB_SK_LDQ ".v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                     : "l"(p));
    }
    return r;
}
__device__ __forceinline__ float ldg_stream_f1(const float* p) {
    float r;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ void sts128(float* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(a), "r"(b),
                 "r"(c), "r"(d)
                 : "memory");
}

// max.NaN: propagates NaN so one instruction checks both range and NaN/Inf.
__device__ __forceinline__ float fmax_nan_abs(float a, float q) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(fabsf(q)));
    return r;
}

// Shared-memory layout (plan tables are loaded once per persistent CTA):
//   T    [Q4*CW + 64] fp32  staged tile of 32 points (see above); words Q4*CW.. stay 0
//   pairs[2m]  u32          byte offsets of each bin's first two coordinates (zero slot if missing)
//   coff [m]   fp32         b_l / w
//   bp   [m+1] u32          first bin-sorted index of every bin
//   cnt  [m]   u8           (unused by the kernel body; kept for the layout's users)
//   ent  [d]   u16          T word offset of the coordinate at each bin-sorted index
//   sgn  [ceil(d/32)] u32   bit j set: sign(j) = -1
//   fold [L+1+d] u32        fold_ptr[L+1], then the fold entries (dst word << 16 | src word)
struct SketchSmem {
    size_t t, bp, cnt, ent, coff, sgn, pairs, fold, total;
};
__host__ __device__ inline SketchSmem sketch_smem_layout(int Q, int m, int d, int L) {
    SketchSmem o{};
    size_t x = 0;
    o.t = x;
    x += ((size_t)(Q / 4) * CW + 64) * 4;
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
    o.fold = x;
    x += (size_t)(L + 1 + d) * 4;   // at most d - 2 fold entries
    o.total = (x + 15) / 16 * 16;
    return o;
}

// Q4 = float4 columns per staged row (16, 64, 256: d <= 64, 256, 1024).
// VEC: 128-bit staging (d % 4 == 0, ld % 4 == 0, 16-byte aligned X); else scalar.
// KT > 0: keys-only hot path for K == KT (pair gathers, biased fast floor);
// KT == 0: any K, and the debug outputs (codes / bits / proj).
template <int Q4, bool VEC, int KT, bool E2>
__global__ void __launch_bounds__(kThreads, 1)
    sketch_kernel(SketchPlanDev plan, DiscretizeDev dz, const float* __restrict__ X, int64_t n, int64_t ld,
                  HashOut out, int dbg) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int Q = 4 * Q4;
    constexpr int NG = kThreads / Q4;                 // row-group slots (4 rows each) per pass of the CTA
    constexpr int RG = NG >= 8 ? 1 : 8 / NG;          // row groups per thread (VEC)
    constexpr int VS = Q4 >= 16 ? Q4 / 16 : 1;        // float4 per thread (scalar staging)
    constexpr uint32_t ZW = (uint32_t)Q4 * CW;
    static_assert(KT == 0 || VEC, "the keys-only path stages with 128-bit loads");
    const int m = plan.m, L = plan.L, d = plan.d;
    const int K = KT > 0 ? KT : plan.K;
    const SketchSmem so = sketch_smem_layout(Q, m, d, L);
    float* T = reinterpret_cast<float*>(smem_raw + so.t);
    uint32_t* s_bp = reinterpret_cast<uint32_t*>(smem_raw + so.bp);
    uint16_t* s_ent = reinterpret_cast<uint16_t*>(smem_raw + so.ent);
    float* s_coff = reinterpret_cast<float*>(smem_raw + so.coff);
    uint32_t* s_sgn = reinterpret_cast<uint32_t*>(smem_raw + so.sgn);
    uint32_t* s_pairs = reinterpret_cast<uint32_t*>(smem_raw + so.pairs);
    uint32_t* s_fptr = reinterpret_cast<uint32_t*>(smem_raw + so.fold);
    uint32_t* s_fold = s_fptr + L + 1;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = (n + 31) >> 5;
    int64_t tile = blockIdx.x;
    if (tile >= ntiles) return;

    for (int i = tid; i <= m; i += kThreads) s_bp[i] = __ldg(plan.bin_ptr + i);
    for (int i = tid; i < m; i += kThreads) {
        s_coff[i] = E2 ? __ldg(dz.c_off + i) : 0.f;
        s_pairs[2 * i] = __ldg(plan.pairs + 2 * i);
        s_pairs[2 * i + 1] = __ldg(plan.pairs + 2 * i + 1);
    }
    for (int i = tid; i < d; i += kThreads) s_ent[i] = __ldg(plan.pos + i);
    for (int i = tid; i < (d + 31) / 32; i += kThreads) s_sgn[i] = __ldg(plan.sign_bits + i);
    for (int i = tid; i <= L; i += kThreads) s_fptr[i] = __ldg(plan.fold_ptr + i);
    for (int i = tid; i < plan.nfold; i += kThreads) s_fold[i] = __ldg(plan.fold + i);
    for (int i = tid; i < 64; i += kThreads) T[ZW + i] = 0.f;
    __syncthreads();

    // VEC: this thread's float4 column c and row groups rg, rg + NG, ...
    const int c = tid % Q4, rg = tid / Q4;
    const bool col_ok = VEC && 4 * c < d && rg < 8;
    uint32_t sm[4] = {0u, 0u, 0u, 0u};
    if (col_ok) {
        const uint32_t w = s_sgn[(4 * c) >> 5] >> ((4 * c) & 31);  // 4 | 4c: never straddles a word
#pragma unroll
        for (int j = 0; j < 4; ++j) sm[j] = ((w >> j) & 1u) << 31;
    }
    float4 buf[VEC ? RG * 4 : VS];

    // row groups [i0, i1) of the thread's column (VEC); the scalar path ignores them
    constexpr bool kEF = LSHB_SK_LDHINT == 2 || LSHB_SK_LDHINT == 3 || (LSHB_SK_LDHINT == 4 && E2);
    auto load = [&](int64_t tl, int i0 = 0, int i1 = 1 << 20) {
        if constexpr (VEC) {
            if (col_ok) {
#pragma unroll
                for (int i = 0; i < RG; ++i) {
                    if (i < i0 || i >= i1) continue;
                    const int64_t r = tl * 32 + 4 * (rg + NG * i);
                    const float* src = X + r * ld + 4 * c;
                    if (tl * 32 + 32 <= n) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) buf[4 * i + j] = ldg_stream_f4<kEF>(src + j * ld);
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            buf[4 * i + j] = r + j < n ? ldg_stream_f4<kEF>(src + j * ld) : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
            }
        } else {
#pragma unroll
            for (int v = 0; v < VS; ++v) {
                float e[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int f = tid + kThreads * (4 * v + q);
                    const int r = f / Q, k = f % Q;
                    const int64_t row = tl * 32 + r;
                    e[q] = (r < 32 && row < n && k < d) ? ldg_stream_f1(X + row * ld + k) : 0.f;
                }
                buf[v] = make_float4(e[0], e[1], e[2], e[3]);
            }
        }
    };
    auto store = [&](int i0 = 0, int i1 = 1 << 20) {
        if constexpr (VEC) {
            if (col_ok) {
#pragma unroll
                for (int i = 0; i < RG; ++i) {
                    if (i < i0 || i >= i1) continue;
                    float* dst = T + c * CW + 4 * (rg + NG * i);
                    const float4 a = buf[4 * i], b = buf[4 * i + 1], cc = buf[4 * i + 2], e = buf[4 * i + 3];
                    sts128(dst, __float_as_uint(a.x) ^ sm[0], __float_as_uint(b.x) ^ sm[0],
                           __float_as_uint(cc.x) ^ sm[0], __float_as_uint(e.x) ^ sm[0]);
                    sts128(dst + 32, __float_as_uint(a.y) ^ sm[1], __float_as_uint(b.y) ^ sm[1],
                           __float_as_uint(cc.y) ^ sm[1], __float_as_uint(e.y) ^ sm[1]);
                    sts128(dst + 64, __float_as_uint(a.z) ^ sm[2], __float_as_uint(b.z) ^ sm[2],
                           __float_as_uint(cc.z) ^ sm[2], __float_as_uint(e.z) ^ sm[2]);
                    sts128(dst + 96, __float_as_uint(a.w) ^ sm[3], __float_as_uint(b.w) ^ sm[3],
                           __float_as_uint(cc.w) ^ sm[3], __float_as_uint(e.w) ^ sm[3]);
                }
            }
        } else {
#pragma unroll
            for (int v = 0; v < VS; ++v) {
                const float e[4] = {buf[v].x, buf[v].y, buf[v].z, buf[v].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int f = tid + kThreads * (4 * v + q);
                    const int r = f / Q, k = f % Q;
                    if (r < 32 && k < d) {
                        const uint32_t sg = ((s_sgn[k >> 5] >> (k & 31)) & 1u) << 31;
                        T[(k >> 2) * CW + (k & 3) * 32 + r] = __uint_as_float(__float_as_uint(e[q]) ^ sg);
                    }
                }
            }
        }
    };

    load(tile);
    const float cs = dz.c_scale;
    float* const Tw = T + lane;   // this lane's (point's) column of the staged tile
    const float* Tl = Tw;
    while (true) {
        __syncthreads();  // previous gathers finished with T
        const int64_t ntile = tile + gridDim.x;
        const bool has_next = ntile < ntiles;
        // the next tile's loads go out as soon as their registers are stored (in halves),
        // so HBM stays busy through the staging phase and the barrier
        if constexpr (VEC && RG >= 2) {
            store(0, RG / 2);
            if (has_next) load(ntile, 0, RG / 2);
            store(RG / 2, RG);
            if (has_next) load(ntile, RG / 2, RG);
        } else {
            store();
            if (has_next) load(ntile);
        }
        __syncthreads();   // the loads above are in flight during the gathers below
        const int64_t row = tile * 32 + lane;
        const bool valid = row < n;
#if LSHB_SK_QUAD
        if constexpr (KT > 0 && (E2 || LSHB_SK_QUAD == 2)) {
            // hot path, four tables per warp: lane = (table j = lane / 8, point quad g =
            // lane % 8); a lane sums, discretises and keys points 4g..4g+3 of table
            // 4G + j.  Every gather is ONE 128-bit load of four points' staged word (the
            // staged row of a coordinate is 32 consecutive points), so a quarter-warp
            // reads one whole 128-byte row: conflict-free, and a quarter of the
            // shared-memory instructions and address adds of one gather per point.  The
            // arithmetic per (bin, point) is the lane-per-point path's, in the same order
            // (fold, then the pair sum), so the keys are bit-identical.
            const int j = lane >> 3, g = lane & 7;
            const char* Tg = reinterpret_cast<const char*>(T) + 16 * g;
            const int64_t row0 = tile * 32 + 4 * g;
            for (int G = warp; 4 * G < L; G += kWarps) {
                const bool tv = 4 * G + j < L;
                const int t = tv ? 4 * G + j : L - 1;   // a clamped lane computes, never folds or stores
                const uint4* pp4 = reinterpret_cast<const uint4*>(s_pairs + t * KT * 2);
                // the first pair offsets are read before the fold (their latency overlaps it)
                constexpr int NPRE = LSHB_SK_QPRE < KT / 2 ? LSHB_SK_QPRE : KT / 2;
                uint4 pv[NPRE > 0 ? NPRE : 1];
#pragma unroll
                for (int i = 0; i < NPRE; ++i) pv[i] = pp4[i];
                {
                    const uint32_t f1 = tv ? s_fptr[t + 1] : 0u;
#pragma unroll 1
                    for (uint32_t f = tv ? s_fptr[t] : 0u; f < f1; ++f) {
                        const uint32_t e = s_fold[f];
                        float4* dst = reinterpret_cast<float4*>(const_cast<char*>(Tg) + 4 * (e >> 16));
                        const float4 b = *reinterpret_cast<const float4*>(Tg + 4 * (e & 0xffffu));
                        float4 a = *dst;
                        a.x += b.x;
                        a.y += b.y;
                        a.z += b.z;
                        a.w += b.w;
                        *dst = a;
                    }
                }
                uint64_t f[4];
                if constexpr (E2) {
                    FpKey fk[4];
                    float qmax = 0.f;
                    const float4* co = reinterpret_cast<const float4*>(s_coff + t * KT);
#pragma unroll
                    for (int k4 = 0; k4 < KT / 4; ++k4) {
                        const float4 c4v = co[k4];
                        const float cc[4] = {c4v.x, c4v.y, c4v.z, c4v.w};
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const uint4 v = 2 * k4 + h < NPRE ? pv[(2 * k4 + h) % (NPRE > 0 ? NPRE : 1)] : pp4[2 * k4 + h];
                            const float4 a0 = *reinterpret_cast<const float4*>(Tg + v.x);
                            const float4 a1 = *reinterpret_cast<const float4*>(Tg + v.y);
                            const float4 b0 = *reinterpret_cast<const float4*>(Tg + v.z);
                            const float4 b1 = *reinterpret_cast<const float4*>(Tg + v.w);
                            const float ya[4] = {a0.x + a1.x, a0.y + a1.y, a0.z + a1.z, a0.w + a1.w};
                            const float yb[4] = {b0.x + b1.x, b0.y + b1.y, b0.z + b1.z, b0.w + b1.w};
#pragma unroll
                            for (int p = 0; p < 4; ++p) {
                                const float qa = fmaf(ya[p], cs, cc[2 * h]);
                                const float qb = fmaf(yb[p], cs, cc[2 * h + 1]);
                                qmax = fmax_nan_abs(fmax_nan_abs(qmax, qa), qb);
                                fk[p].add(__float_as_uint(__fadd_rd(qa, 12582912.0f)));
                                fk[p].add(__float_as_uint(__fadd_rd(qb, 12582912.0f)));
                            }
                        }
                    }
                    if (qmax < 4194304.0f) {
#pragma unroll
                        for (int p = 0; p < 4; ++p) fk[p].unbias(KT);
                    } else {
                        // rare: a code outside the fast floor range (or NaN/Inf) in one of the
                        // lane's four points: redo all four exactly
#pragma unroll
                        for (int p = 0; p < 4; ++p) fk[p] = FpKey();
#pragma unroll 1
                        for (int kk = 0; kk < KT; ++kk) {
                            const uint32_t o1 = s_pairs[2 * (t * KT + kk)], o2 = s_pairs[2 * (t * KT + kk) + 1];
                            const float c0 = s_coff[t * KT + kk];
#pragma unroll
                            for (int p = 0; p < 4; ++p) {
                                const float y = *reinterpret_cast<const float*>(Tg + o1 + 4 * p) +
                                                *reinterpret_cast<const float*>(Tg + o2 + 4 * p);
                                fk[p].add((uint32_t)floor_code(fmaf(y, cs, c0), dz.flags));
                            }
                        }
                    }
#pragma unroll
                    for (int p = 0; p < 4; ++p) f[p] = fk[p].key();
                } else {
                    uint32_t sb[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                    for (int i = 0; i < KT / 2; ++i) {
                        const uint4 v = i < NPRE ? pv[i % (NPRE > 0 ? NPRE : 1)] : pp4[i];
                        const float4 a0 = *reinterpret_cast<const float4*>(Tg + v.x);
                        const float4 a1 = *reinterpret_cast<const float4*>(Tg + v.y);
                        const float4 b0 = *reinterpret_cast<const float4*>(Tg + v.z);
                        const float4 b1 = *reinterpret_cast<const float4*>(Tg + v.w);
                        const float ya[4] = {a0.x + a1.x, a0.y + a1.y, a0.z + a1.z, a0.w + a1.w};
                        const float yb[4] = {b0.x + b1.x, b0.y + b1.y, b0.z + b1.z, b0.w + b1.w};
#pragma unroll
                        for (int p = 0; p < 4; ++p)
                            sb[p] |= (ya[p] > 0.0f ? 1u : 0u) << (2 * i) | (yb[p] > 0.0f ? 1u : 0u) << (2 * i + 1);
                    }
#pragma unroll
                    for (int p = 0; p < 4; ++p) f[p] = sb[p];
                }
                if (tv && out.keys) {
                    uint64_t* kp = out.keys + (int64_t)t * n + row0;
#if LSHB_SK_ST128 >= 2
                    if (row0 + 4 <= n && (reinterpret_cast<uintptr_t>(kp) & 31) == 0) {
#if LSHB_SK_ST128 == 3
                        asm volatile("st.global.cs.v4.b64 [%0], {%1,%2,%3,%4};" ::"l"(kp), "l"(f[0]), "l"(f[1]), "l"(f[2]),
                                     "l"(f[3])
                                     : "memory");
#else
                        asm volatile("st.global.v4.b64 [%0], {%1,%2,%3,%4};" ::"l"(kp), "l"(f[0]), "l"(f[1]), "l"(f[2]),
                                     "l"(f[3])
                                     : "memory");
#endif
                    } else
#endif
#if LSHB_SK_ST128
                    if (row0 + 4 <= n && (reinterpret_cast<uintptr_t>(kp) & 15) == 0) {
                        reinterpret_cast<ulonglong2*>(kp)[0] = make_ulonglong2(f[0], f[1]);
                        reinterpret_cast<ulonglong2*>(kp)[1] = make_ulonglong2(f[2], f[3]);
                    } else
#endif
#pragma unroll
                    for (int p = 0; p < 4; ++p)
                        if (row0 + p < n && LSHB_OK(row0 + p < n)) kp[p] = f[p];
                }
            }
        } else
#endif
        if constexpr (KT > 0) {
            // hot path: the 3rd, 4th, ... coordinates of a bin are first folded into its
            // first coordinate's staged word (this lane's own column: no other lane or warp
            // reads it — a coordinate belongs to one bin, a bin to one table, a table to one
            // warp); then every bin is the sum of two staged words through `pairs`
            // (branch-free; a missing one reads the zero slot).  Two tables per iteration.
#pragma unroll kTUnroll
            for (int t = warp; t < L; t += kWarps) {
                float acc[KT];
                {
                    const uint32_t f1 = s_fptr[t + 1];
#pragma unroll 1
                    for (uint32_t f = s_fptr[t]; f < f1; ++f) {
                        const uint32_t e = s_fold[f];
                        Tw[e >> 16] += Tw[e & 0xffffu];
                    }
                }
                {
                    // two byte offsets per bin, 2 bins per 128-bit load; one add each
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
                uint64_t f;
                if constexpr (E2) {
                    // fast floor: the fp32 bits of q + 1.5*2^23 (rounded toward -inf) are
                    // LSHB_FLOOR_BIAS + floor(q) for |q| < 2^22; both Horner lanes take those
                    // biased words and drop the bias once per table (FpKey::unbias)
                    FpKey fk;
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
                            fk.add(__float_as_uint(__fadd_rd(q, 12582912.0f)));
                        }
                    }
                    if (qmax < 4194304.0f) {
                        fk.unbias(KT);
                    } else {
                        // rare: a code outside the fast floor range (or NaN/Inf): redo exactly
                        fk = FpKey();
#pragma unroll
                        for (int kk = 0; kk < KT; ++kk)
                            fk.add((uint32_t)floor_code(fmaf(acc[kk], cs, s_coff[t * KT + kk]), dz.flags));
                    }
                    f = fk.key();
                } else {
                    uint32_t sb = 0;
#pragma unroll
                    for (int kk = 0; kk < KT; ++kk) sb |= (acc[kk] > 0.0f ? 1u : 0u) << kk;
                    f = sb;
                }
                if (valid && out.keys && LSHB_OK(row < n)) out.keys[(int64_t)t * n + row] = f;
            }
        } else {
            // generic K (and the debug outputs): sequential sum over each bin's coordinates
            for (int t = warp; t < L; t += kWarps) {
                uint64_t sbits = 0;
                FpKey fk;
                for (int kk = 0; kk < K; ++kk) {
                    const int l = t * K + kk;
                    // ((x_1 + x_3) + x_4 + ...) + x_2 in bin-sorted order: the fast path's fold order
                    const uint32_t j0 = s_bp[l], j1 = s_bp[l + 1];
                    float acc = 0.0f;
                    if (j1 > j0) acc += Tl[s_ent[j0]];
                    for (uint32_t j = j0 + 2; j < j1; ++j) acc += Tl[s_ent[j]];
                    if (j1 > j0 + 1) acc += Tl[s_ent[j0 + 1]];
                    int32_t z;
                    if constexpr (E2) {
                        z = floor_code(fmaf(acc, cs, s_coff[l]), dz.flags);
                        fk.add((uint32_t)z);
                    } else {
                        z = acc > 0.0f ? 1 : 0;
                        sbits |= (uint64_t)z << kk;
                    }
                    if (dbg && valid) {
                        if (out.proj) out.proj[row * m + l] = acc;
                        if (E2 && out.codes) out.codes[row * m + l] = z;
                        if (!E2 && out.bits && z) atomicOr(&out.bits[row * ((m + 31) >> 5) + (l >> 5)], 1u << (l & 31));
                    }
                }
                if (valid && out.keys && LSHB_OK(row < n)) out.keys[(int64_t)t * n + row] = E2 ? fk.key() : sbits;
            }
        }
        if (!has_next) break;
        tile = ntile;
    }
}

template <int Q4, bool VEC, int KT, bool E2>
cudaError_t launch_t(const SketchPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n, int64_t ld,
                     HashOut out, int num_sms, cudaStream_t s) {
    const size_t smem = sketch_smem_layout(4 * Q4, plan.m, plan.d, plan.L).total;
    auto kern = sketch_kernel<Q4, VEC, KT, E2>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = (n + 31) / 32;
    const int grid = (int)(ntiles < num_sms ? ntiles : num_sms);
    const int dbg = (out.codes || out.bits || out.proj) ? 1 : 0;
    kern<<<grid, kThreads, smem, s>>>(plan, dz, X, n, ld, out, dbg);
    return cudaGetLastError();
}

}  // namespace sk
}  // namespace lshb
