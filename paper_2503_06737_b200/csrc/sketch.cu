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
//   T    [(Q+2) x 33] fp32  staged chunk of 32 points: coordinate k of point r lives at
//                           word pos(k)*33 + r, pos = rank of k in bin-sorted order, value
//                           already multiplied by sign(k); so every bin is a run of
//                           consecutive positions and lane r reads word p*33 + r
//                           (bank-conflict free).  +2 positions: branch-free over-read.
//   ys   [m x 32]  fp32     partial bins across chunks (multi-chunk plans only)
//   bp   [nchunks x (m+1)]  first position (absolute coordinate index) of every bin
//   cnt  [nchunks x m] u8   coordinates per bin per chunk (saturated at 255)
//   pos  [d] u16            bin-sorted position of coordinate j inside its chunk
//   coff [m] fp32           b_l / w
//   sgn  [ceil(d/32)] u32   bit j set: sign(j) = -1
__host__ __device__ inline size_t sketch_smem_layout(int Q, int m, int d, int nchunks, size_t* o_ys, size_t* o_bp,
                                                     size_t* o_cnt, size_t* o_pos, size_t* o_coff, size_t* o_sgn) {
    size_t o = (size_t)(Q + 2) * 33 * 4;
    *o_ys = o;
    if (nchunks > 1) o += (size_t)m * 32 * 4;
    *o_bp = o;
    o += (size_t)nchunks * (m + 1) * 4;
    *o_cnt = o = (o + 15) / 16 * 16;
    o += ((size_t)nchunks * m + 15) / 16 * 16;
    *o_pos = o;
    o += ((size_t)d * 2 + 15) / 16 * 16;
    *o_coff = o;
    o += (size_t)m * 4;
    *o_sgn = o;
    o += (size_t)((d + 31) / 32) * 4;
    return o;
}

// max.NaN: propagates NaN so one instruction checks both range and NaN/Inf.
__device__ __forceinline__ float fmax_nan_abs(float a, float q) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(fabsf(q)));
    return r;
}

template <int VPT, bool VEC, int KT, bool E2, bool SINGLE>
__global__ void __launch_bounds__(kThreads, 1)
    sketch_kernel(SketchPlanDev plan, DiscretizeDev dz, const float* __restrict__ X, int64_t n, int64_t ld,
                  HashOut out, int dbg) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int Q = 64 * VPT;
    constexpr int Q4 = Q / 4;                 // float4 per row of a chunk
    constexpr int RPI = kThreads / Q4;        // rows per load iteration (VEC path)
    const int m = plan.m, L = plan.L, d = plan.d, nch = plan.nchunks;
    const int K = KT > 0 ? KT : plan.K;
    size_t o_ys, o_bp, o_cnt, o_pos, o_coff, o_sgn;
    sketch_smem_layout(Q, m, d, nch, &o_ys, &o_bp, &o_cnt, &o_pos, &o_coff, &o_sgn);
    float* T = reinterpret_cast<float*>(smem_raw);
    float* ys = reinterpret_cast<float*>(smem_raw + o_ys);
    uint32_t* s_bp = reinterpret_cast<uint32_t*>(smem_raw + o_bp);
    uint8_t* s_cnt = reinterpret_cast<uint8_t*>(smem_raw + o_cnt);
    uint16_t* s_pos = reinterpret_cast<uint16_t*>(smem_raw + o_pos);
    float* s_coff = reinterpret_cast<float*>(smem_raw + o_coff);
    uint32_t* s_sgn = reinterpret_cast<uint32_t*>(smem_raw + o_sgn);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = (n + 31) >> 5;
    int64_t tile = blockIdx.x;
    if (tile >= ntiles) return;

    for (int i = tid; i < nch * (m + 1); i += kThreads) s_bp[i] = __ldg(plan.bin_ptr + i);
    for (int i = tid; i < nch * m; i += kThreads) {
        const int cc = i / m, l = i % m;
        const uint32_t cn = __ldg(plan.bin_ptr + cc * (m + 1) + l + 1) - __ldg(plan.bin_ptr + cc * (m + 1) + l);
        s_cnt[i] = (uint8_t)(cn < 255u ? cn : 255u);
    }
    for (int i = tid; i < d; i += kThreads) s_pos[i] = __ldg(plan.pos + i);
    for (int i = tid; i < m; i += kThreads) s_coff[i] = E2 ? __ldg(dz.c_off + i) : 0.f;
    for (int i = tid; i < (d + 31) / 32; i += kThreads) s_sgn[i] = __ldg(plan.sign_bits + i);
    for (int i = tid; i < 2 * 33; i += kThreads) T[Q * 33 + i] = 0.f;
    __syncthreads();

    float4 buf[VPT];
    // staging targets of this thread's 4 columns (VEC path): word offset pos*33, sign mask
    uint32_t so[4] = {0, 0, 0, 0}, sm[4] = {0, 0, 0, 0};
    bool col_ok = false;
    auto columns_for_chunk = [&](int c) {
        if constexpr (VEC) {
            const int k = c * Q + 4 * (tid % Q4);
            col_ok = k < d;
            if (col_ok) {
                const uint32_t w = s_sgn[k >> 5] >> (k & 31);  // 4 | k: never straddles a word
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    so[e] = (uint32_t)s_pos[k + e] * 33u;
                    sm[e] = ((w >> e) & 1u) << 31;
                }
            }
        }
    };

    auto load = [&](int64_t tl, int c) {
        const int k0 = c * Q;
        const int Qc = min(Q, d - k0);
        if constexpr (VEC) {
            const int r0 = tid / Q4, c4 = tid % Q4;
            if (4 * c4 < Qc) {
                const float* src = X + (tl * 32 + r0) * ld + k0 + 4 * c4;
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
                    e[q] = (row < n && k < Qc) ? ldg_stream_f1(X + row * ld + k0 + k) : 0.f;
                }
                buf[v] = make_float4(e[0], e[1], e[2], e[3]);
            }
        }
    };
    auto store = [&](int c) {
        if constexpr (VEC) {
            if (col_ok) {
                const int r0 = tid / Q4;
#pragma unroll
                for (int v = 0; v < VPT; ++v) {
                    const int r = r0 + v * RPI;
                    T[so[0] + r] = __uint_as_float(__float_as_uint(buf[v].x) ^ sm[0]);
                    T[so[1] + r] = __uint_as_float(__float_as_uint(buf[v].y) ^ sm[1]);
                    T[so[2] + r] = __uint_as_float(__float_as_uint(buf[v].z) ^ sm[2]);
                    T[so[3] + r] = __uint_as_float(__float_as_uint(buf[v].w) ^ sm[3]);
                }
            }
        } else {
            const int k0 = c * Q;
            const int Qc = min(Q, d - k0);
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                const float e[4] = {buf[v].x, buf[v].y, buf[v].z, buf[v].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int f = tid + kThreads * (4 * v + q);
                    const int r = f / Q, k = f % Q;
                    if (k < Qc) {
                        const int kg = k0 + k;
                        const uint32_t sg = ((s_sgn[kg >> 5] >> (kg & 31)) & 1u) << 31;
                        T[(uint32_t)s_pos[kg] * 33u + r] = __uint_as_float(__float_as_uint(e[q]) ^ sg);
                    }
                }
            }
        }
    };

    int c = 0;
    columns_for_chunk(0);
    load(tile, 0);
    const float cs = dz.c_scale;
    while (true) {
        __syncthreads();  // previous gathers finished with T
        store(c);
        __syncthreads();
        int64_t ntile = tile;
        int nc = c + 1;
        if (nc == nch) {
            nc = 0;
            ntile += gridDim.x;
        }
        const bool has_next = ntile < ntiles;
        if (has_next) load(ntile, nc);  // in flight during the gathers below
        if constexpr (!SINGLE) columns_for_chunk(nc);

        const bool first = SINGLE || c == 0, last = SINGLE || c == nch - 1;
        const int64_t row = tile * 32 + lane;
        const bool valid = row < n;
        const uint32_t* bpc = s_bp + (SINGLE ? 0 : c * (m + 1));
        const uint8_t* cntc = s_cnt + (SINGLE ? 0 : (size_t)c * m);
        const uint32_t cbase = SINGLE ? 0u : (uint32_t)(c * Q);
        if constexpr (KT > 0 && SINGLE) {
            // Phased table loop (hot path): all 2*K loads first (branch-free for bins with
            // <= 2 coordinates), rare fix-ups for fuller bins, then discretise + key.
            for (int t = warp; t < L; t += kWarps) {
                const float* p = T + bpc[t * K] * 33 + lane;
                uint32_t cw[KT / 4];
                const uint32_t* cp = reinterpret_cast<const uint32_t*>(cntc + t * KT);
#pragma unroll
                for (int i = 0; i < KT / 4; ++i) cw[i] = cp[i];
                float acc[KT];
                uint32_t big = 0;
                {
                    const float* pp = p;
#pragma unroll
                    for (int kk = 0; kk < KT; ++kk) {
                        const uint32_t cnt = (cw[kk >> 2] >> (8 * (kk & 3))) & 255u;
                        const float v0 = pp[0];
                        const float v1 = pp[33];
                        float a = cnt > 0 ? 0.0f + v0 : 0.0f;
                        a = cnt > 1 ? a + v1 : a;
                        acc[kk] = a;
                        big |= (cnt > 2 ? 1u : 0u) << kk;
                        pp += cnt * 33;
                    }
                }
                if (big) {
                    const float* pp = p;
#pragma unroll
                    for (int kk = 0; kk < KT; ++kk) {
                        const uint32_t cnt = (cw[kk >> 2] >> (8 * (kk & 3))) & 255u;
                        if (cnt > 2)
                            for (uint32_t j = 2; j < cnt; ++j) acc[kk] += pp[j * 33];
                        pp += cnt * 33;
                    }
                }
                uint64_t f = E2 ? LSHB_FNV_OFFSET : 0ull;
                if constexpr (E2) {
                    float qmax = 0.f;
                    const float4* co = reinterpret_cast<const float4*>(s_coff + t * KT);
#pragma unroll
                    for (int k4 = 0; k4 < KT / 4; ++k4) {
                        const float4 c4 = co[k4];
                        const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float q = fmaf(acc[4 * k4 + j], cs, cc[j]);
                            qmax = fmax_nan_abs(qmax, q);
                            const int32_t z = __float_as_int(__fadd_rd(q, 12582912.0f)) - 0x4B400000;
                            f = (f ^ (uint64_t)(uint32_t)z) * LSHB_FNV_PRIME;
                        }
                    }
                    if (!(qmax < 4194304.0f)) {
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
        } else
        for (int t = warp; t < L; t += kWarps) {
            const float* p = T + (bpc[t * K] - cbase) * 33 + lane;
            uint64_t f = E2 ? LSHB_FNV_OFFSET : 0ull;
            uint32_t sbits = 0;
            float qmax = 0.f;
            // one bin: y = sum of its (sign-applied) coordinates in ascending coordinate order
            auto bin = [&](int kk, uint32_t cnt) {
                const int l = t * K + kk;
                float acc = first ? 0.0f : ys[l * 32 + lane];
                const float v0 = p[0];
                const float v1 = p[33];
                if (cnt <= 2) {                      // m ~ d: 0..2 coordinates per bin, branch-free
                    acc = cnt > 0 ? acc + v0 : acc;
                    acc = cnt > 1 ? acc + v1 : acc;
                } else {
                    acc = (acc + v0) + v1;
                    for (uint32_t j = 2; j < cnt; ++j) acc += p[j * 33];
                }
                p += cnt * 33;
                if (!last) {
                    ys[l * 32 + lane] = acc;
                    return;
                }
                int32_t z;
                if constexpr (E2) {
                    const float q = fmaf(acc, cs, s_coff[l]);
                    qmax = fmax_nan_abs(qmax, q);
                    z = __float_as_int(__fadd_rd(q, 12582912.0f)) - 0x4B400000;  // floor(q), |q| < 2^22
                    f = (f ^ (uint64_t)(uint32_t)z) * LSHB_FNV_PRIME;
                } else {
                    z = acc > 0.0f ? 1 : 0;
                    if (KT > 0 && KT <= 32) sbits |= (uint32_t)z << kk;
                    else f |= (uint64_t)z << kk;
                }
                if (KT == 0 && dbg && valid) {  // debug outputs only in the generic instantiation
                    if (out.proj) out.proj[row * m + l] = acc;
                    if (E2 && out.codes) out.codes[row * m + l] = z;
                    if (!E2 && out.bits && z) atomicOr(&out.bits[row * ((m + 31) >> 5) + (l >> 5)], 1u << (l & 31));
                }
            };
            if constexpr (KT > 0) {
                uint32_t cw[KT / 4];
                const uint32_t* cp = reinterpret_cast<const uint32_t*>(cntc + t * KT);
#pragma unroll
                for (int i = 0; i < KT / 4; ++i) cw[i] = cp[i];
#pragma unroll
                for (int kk = 0; kk < KT; ++kk) bin(kk, (cw[kk >> 2] >> (8 * (kk & 3))) & 255u);
            } else {
                for (int kk = 0; kk < K; ++kk) bin(kk, bpc[t * K + kk + 1] - bpc[t * K + kk]);
            }
            if (!last) continue;
            if constexpr (E2) {
                if (!(qmax < 4194304.0f)) {
                    // rare: a code outside the fast floor range (or NaN/Inf): redo this table exactly
                    f = LSHB_FNV_OFFSET;
                    const float* p2 = T + (bpc[t * K] - cbase) * 33 + lane;
                    for (int kk = 0; kk < K; ++kk) {
                        const int l = t * K + kk;
                        float acc = first ? 0.0f : ys[l * 32 + lane];
                        const uint32_t cnt = bpc[l + 1] - bpc[l];
                        for (uint32_t j = 0; j < cnt; ++j) acc += p2[j * 33];
                        p2 += cnt * 33;
                        const int32_t z = floor_code(fmaf(acc, cs, s_coff[l]), dz.flags);
                        f = (f ^ (uint64_t)(uint32_t)z) * LSHB_FNV_PRIME;
                        if (KT == 0 && dbg && valid && out.codes) out.codes[row * m + l] = z;
                    }
                }
            } else if (KT > 0 && KT <= 32) {
                f = sbits;
            }
            if (valid && out.keys) out.keys[(int64_t)t * n + row] = E2 ? fmix64_dev(f) : f;
        }
        if (!has_next) break;
        tile = ntile;
        c = nc;
    }
}

size_t sketch_smem_bytes(int Q, int m, int d, int nchunks) {
    size_t a, b, c, e, f, g;
    return sketch_smem_layout(Q, m, d, nchunks, &a, &b, &c, &e, &f, &g);
}

template <int VPT, bool VEC, int KT, bool E2, bool SINGLE>
static cudaError_t launch_t(const SketchPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n, int64_t ld,
                            HashOut out, int num_sms, cudaStream_t s) {
    const size_t smem = sketch_smem_bytes(64 * VPT, plan.m, plan.d, plan.nchunks);
    auto kern = sketch_kernel<VPT, VEC, KT, E2, SINGLE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = (n + 31) / 32;
    const int grid = (int)(ntiles < num_sms ? ntiles : num_sms);
    const int dbg = (out.codes || out.bits || out.proj) ? 1 : 0;
    kern<<<grid, kThreads, smem, s>>>(plan, dz, X, n, ld, out, dbg);
    return cudaGetLastError();
}

template <int VPT, bool VEC, bool SINGLE>
static cudaError_t launch_k(const SketchPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n, int64_t ld,
                            HashOut out, int num_sms, cudaStream_t s) {
    const bool e2 = dz.e2lsh != 0;
    const bool dbg = out.codes || out.bits || out.proj;  // debug outputs: generic instantiation
    if (plan.K == 16 && plan.max_cnt <= 255 && !dbg)
        return e2 ? launch_t<VPT, VEC, 16, true, SINGLE>(plan, dz, X, n, ld, out, num_sms, s)
                  : launch_t<VPT, VEC, 16, false, SINGLE>(plan, dz, X, n, ld, out, num_sms, s);
    if (plan.K == 8 && plan.max_cnt <= 255 && !dbg)
        return e2 ? launch_t<VPT, VEC, 8, true, SINGLE>(plan, dz, X, n, ld, out, num_sms, s)
                  : launch_t<VPT, VEC, 8, false, SINGLE>(plan, dz, X, n, ld, out, num_sms, s);
    return e2 ? launch_t<VPT, VEC, 0, true, SINGLE>(plan, dz, X, n, ld, out, num_sms, s)
              : launch_t<VPT, VEC, 0, false, SINGLE>(plan, dz, X, n, ld, out, num_sms, s);
}

cudaError_t launch_sketch(const SketchPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n, int64_t ld,
                          HashOut out, int num_sms, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const bool vec = (plan.d % 4 == 0) && (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
    const bool single = plan.nchunks == 1;
    switch (plan.vpt) {
        case 1:
            return vec ? launch_k<1, true, true>(plan, dz, X, n, ld, out, num_sms, s)
                       : launch_k<1, false, true>(plan, dz, X, n, ld, out, num_sms, s);
        case 4:
            return vec ? launch_k<4, true, true>(plan, dz, X, n, ld, out, num_sms, s)
                       : launch_k<4, false, true>(plan, dz, X, n, ld, out, num_sms, s);
        case 16:
            if (!single) return cudaErrorInvalidValue;  // multi-chunk plans run sketch_chunked.cu
            return vec ? launch_k<16, true, true>(plan, dz, X, n, ld, out, num_sms, s)
                       : launch_k<16, false, true>(plan, dz, X, n, ld, out, num_sms, s);
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
