// sketch_chunked.cu — K1 for plans that do not fit one resident chunk: large d
// and/or large m (C3 CS/HCS with d = 4096, C5 HCS with d = 65536, m = 4096).
//
// Same arithmetic as sketch.cu (Def. CS, Def. HCS PAPER.md:212-215,
// discretisation PAPER.md:314/:624/:918/:1441, keys B1/B10).  The host planner
// splits the L tables into GROUPS whose bins fit the shared-memory partial-sum
// buffer, and streams, per group, exactly the coordinates whose bin falls in the
// group, in CHUNKS of <= 1024 coordinates.  Every coordinate belongs to exactly
// one bin, so X is still read once in total.  For HCS the coordinates of a group
// are whole runs of d_1 contiguous inputs (one (i_2..i_N) per run maps into one
// block of m_1 bins), so the staging loads stay 128-bit and coalesced.
// Within a chunk the coordinates are staged in bin-sorted order with the sign
// applied (as in sketch.cu); partial bin sums persist across the chunks of a group
// in shared memory and the group's tables are discretised on its last chunk.
#include <cuda_runtime.h>
#include <stdint.h>

#include "discretize.cuh"
#include "internal.hpp"

namespace lshb {

namespace {
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int Q = 1024;
constexpr int Q4 = Q / 4;
constexpr int RPI = kThreads / Q4;  // 2 rows per load iteration
constexpr int VPT = 16;

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
__device__ __forceinline__ float fmax_nan_abs_c(float a, float q) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(fabsf(q)));
    return r;
}
}  // namespace

size_t chunked_smem_bytes(int m, int gbins) {
    size_t o = (size_t)(Q + 2) * 33 * 4;        // T
    o += (size_t)gbins * 32 * 4;                // ys
    o += ((size_t)(gbins + 1) * 4 + 15) / 16 * 16;   // bp
    o += ((size_t)(gbins + 1) + 15) / 16 * 16;       // cnt
    o += (size_t)m * 4;                          // coff
    return o;
}

template <bool VEC, int KT, bool E2>
__global__ void __launch_bounds__(kThreads, 1)
    sketch_chunked_kernel(ChunkedPlanDev plan, DiscretizeDev dz, const float* __restrict__ X, int64_t n, int64_t ld,
                          HashOut out, int dbg) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = plan.m, K = KT > 0 ? KT : plan.K, nch = plan.nchunks, GB = plan.gbins;
    float* T = reinterpret_cast<float*>(smem_raw);
    float* ys = T + (Q + 2) * 33;
    uint32_t* s_bp = reinterpret_cast<uint32_t*>(ys + (size_t)GB * 32);
    uint8_t* s_cnt = reinterpret_cast<uint8_t*>(smem_raw + (Q + 2) * 33 * 4 + (size_t)GB * 32 * 4 +
                                                ((size_t)(GB + 1) * 4 + 15) / 16 * 16);
    float* s_coff = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(s_cnt) + ((size_t)(GB + 1) + 15) / 16 * 16);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = (n + 31) >> 5;
    int64_t tile = blockIdx.x;
    if (tile >= ntiles) return;
    for (int i = tid; i < m; i += kThreads) s_coff[i] = E2 ? __ldg(dz.c_off + i) : 0.f;
    for (int i = tid; i < 2 * 33; i += kThreads) T[Q * 33 + i] = 0.f;

    float4 buf[VPT];
    uint32_t so[4] = {0, 0, 0, 0}, sm[4] = {0, 0, 0, 0};
    bool col_ok = false;
    const int r0 = tid / Q4, c4 = tid % Q4;

    auto columns_for_chunk = [&](const ChunkInfoDev& ci) {
        if constexpr (VEC) {
            col_ok = 4 * c4 < ci.Qc;
            if (col_ok) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t k = ci.coord_off + 4 * c4 + e;
                    so[e] = (uint32_t)__ldg(plan.pos + k) * 33u;
                    sm[e] = ((__ldg(plan.sgn + (k >> 5)) >> (k & 31)) & 1u) << 31;
                }
            }
        }
    };
    auto load = [&](int64_t tl, const ChunkInfoDev& ci) {
        if constexpr (VEC) {
            if (4 * c4 < ci.Qc) {
                const int gc = __ldg(plan.gcoord + ci.coord_off + 4 * c4);
                const float* src = X + (tl * 32 + r0) * ld + gc;
                const int64_t stride = (int64_t)RPI * ld;
                if (tl * 32 + 32 <= n) {
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
                    e[q] = (row < n && k < ci.Qc) ? ldg_stream_f1(X + row * ld + __ldg(plan.gcoord + ci.coord_off + k))
                                                   : 0.f;
                }
                buf[v] = make_float4(e[0], e[1], e[2], e[3]);
            }
        }
    };
    auto store = [&](const ChunkInfoDev& ci) {
        if constexpr (VEC) {
            if (col_ok) {
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
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                const float e[4] = {buf[v].x, buf[v].y, buf[v].z, buf[v].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int f = tid + kThreads * (4 * v + q);
                    const int r = f / Q, k = f % Q;
                    if (k < ci.Qc) {
                        const uint32_t kg = ci.coord_off + k;
                        const uint32_t sg = ((__ldg(plan.sgn + (kg >> 5)) >> (kg & 31)) & 1u) << 31;
                        T[(uint32_t)__ldg(plan.pos + kg) * 33u + r] = __uint_as_float(__float_as_uint(e[q]) ^ sg);
                    }
                }
            }
        }
        const int nb = (ci.t1 - ci.t0) * K;
        for (int i = tid; i <= nb; i += kThreads) {
            s_bp[i] = __ldg(plan.bp + ci.bp_off + i);
            s_cnt[i] = __ldg(plan.cnt + ci.bp_off + i);
        }
    };

    int c = 0;
    ChunkInfoDev ci = plan.chunks[0];
    columns_for_chunk(ci);
    load(tile, ci);
    const float cs = dz.c_scale;
    while (true) {
        __syncthreads();  // previous gathers finished with T / bp
        store(ci);
        __syncthreads();
        int64_t ntile = tile;
        int nc = c + 1;
        if (nc == nch) {
            nc = 0;
            ntile += gridDim.x;
        }
        const bool has_next = ntile < ntiles;
        ChunkInfoDev cn = ci;
        if (has_next) {
            cn = plan.chunks[nc];
            load(ntile, cn);  // in flight during the gathers below
        }
        const bool first = ci.flags & 1, last = (ci.flags >> 1) & 1;
        const int64_t row = tile * 32 + lane;
        const bool valid = row < n;
        for (int t = ci.t0 + warp; t < ci.t1; t += kWarps) {
            const int lb0 = (t - ci.t0) * K;
            const float* p = T + s_bp[lb0] * 33 + lane;
            uint64_t f = 0;
            FpKey fk;
            uint32_t sbits = 0;
            float qmax = 0.f;
            auto bin = [&](int kk, uint32_t cnt) {
                const int lb = lb0 + kk, l = t * K + kk;
                float acc = first ? 0.0f : ys[lb * 32 + lane];
                const float v0 = p[0];
                const float v1 = p[33];
                if (cnt <= 2) {
                    acc = cnt > 0 ? acc + v0 : acc;
                    acc = cnt > 1 ? acc + v1 : acc;
                } else {
                    acc = (acc + v0) + v1;
                    for (uint32_t j = 2; j < cnt; ++j) acc += p[j * 33];
                }
                p += cnt * 33;
                if (!last) {
                    ys[lb * 32 + lane] = acc;
                    return;
                }
                int32_t z;
                if constexpr (E2) {
                    const float q = fmaf(acc, cs, s_coff[l]);
                    qmax = fmax_nan_abs_c(qmax, q);
                    z = __float_as_int(__fadd_rd(q, 12582912.0f)) - 0x4B400000;
                    fk.add((uint32_t)z);
                } else {
                    z = acc > 0.0f ? 1 : 0;
                    if (KT > 0 && KT <= 32) sbits |= (uint32_t)z << kk;
                    else f |= (uint64_t)z << kk;
                }
                if (KT == 0 && dbg && valid) {
                    if (out.proj) out.proj[row * m + l] = acc;
                    if (E2 && out.codes) out.codes[row * m + l] = z;
                    if (!E2 && out.bits && z) atomicOr(&out.bits[row * ((m + 31) >> 5) + (l >> 5)], 1u << (l & 31));
                }
            };
            if constexpr (KT > 0) {
#pragma unroll
                for (int kk = 0; kk < KT; ++kk) bin(kk, s_cnt[lb0 + kk]);
            } else {
                for (int kk = 0; kk < K; ++kk) bin(kk, s_bp[lb0 + kk + 1] - s_bp[lb0 + kk]);
            }
            if (!last) continue;
            if constexpr (E2) {
                if (!(qmax < 4194304.0f)) {
                    fk = FpKey();
                    const float* p2 = T + s_bp[lb0] * 33 + lane;
                    for (int kk = 0; kk < K; ++kk) {
                        const int lb = lb0 + kk, l = t * K + kk;
                        float acc = first ? 0.0f : ys[lb * 32 + lane];
                        const uint32_t cnt = s_bp[lb + 1] - s_bp[lb];
                        for (uint32_t j = 0; j < cnt; ++j) acc += p2[j * 33];
                        p2 += cnt * 33;
                        const int32_t z = floor_code(fmaf(acc, cs, s_coff[l]), dz.flags);
                        fk.add((uint32_t)z);
                        if (KT == 0 && dbg && valid && out.codes) out.codes[row * m + l] = z;
                    }
                }
            } else if (KT > 0 && KT <= 32) {
                f = sbits;
            }
            if (valid && out.keys && LSHB_OK(row < n)) out.keys[(int64_t)t * n + row] = E2 ? fk.key() : f;
        }
        if (!has_next) break;
        columns_for_chunk(cn);
        tile = ntile;
        c = nc;
        ci = cn;
    }
}

template <bool VEC, int KT, bool E2>
static cudaError_t launch_c(const ChunkedPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n, int64_t ld,
                            HashOut out, int num_sms, cudaStream_t s) {
    const size_t smem = chunked_smem_bytes(plan.m, plan.gbins);
    auto kern = sketch_chunked_kernel<VEC, KT, E2>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = (n + 31) / 32;
    const int grid = (int)(ntiles < num_sms ? ntiles : num_sms);
    const int dbg = (out.codes || out.bits || out.proj) ? 1 : 0;
    kern<<<grid, kThreads, smem, s>>>(plan, dz, X, n, ld, out, dbg);
    return cudaGetLastError();
}

template <bool VEC>
static cudaError_t launch_ck(const ChunkedPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n,
                             int64_t ld, HashOut out, int num_sms, cudaStream_t s) {
    const bool e2 = dz.e2lsh != 0;
    const bool dbg = out.codes || out.bits || out.proj;
    if (plan.K == 16 && plan.max_cnt <= 255 && !dbg)
        return e2 ? launch_c<VEC, 16, true>(plan, dz, X, n, ld, out, num_sms, s)
                  : launch_c<VEC, 16, false>(plan, dz, X, n, ld, out, num_sms, s);
    return e2 ? launch_c<VEC, 0, true>(plan, dz, X, n, ld, out, num_sms, s)
              : launch_c<VEC, 0, false>(plan, dz, X, n, ld, out, num_sms, s);
}

cudaError_t launch_sketch_chunked(const ChunkedPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n,
                                  int64_t ld, HashOut out, int num_sms, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const bool vec = plan.vec_ok && (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
    return vec ? launch_ck<true>(plan, dz, X, n, ld, out, num_sms, s)
               : launch_ck<false>(plan, dz, X, n, ld, out, num_sms, s);
}

}  // namespace lshb
