// sketch_hcs.cu — K2: the higher-order count sketch (Def. HCS)
// with the Kronecker structure made explicit, fused with discretisation
// (PAPER.md:624 / :1441) and table-key packing (B1, B10).  DESIGN.md §K2.
//
// Structure used (vec(S1 P S2^T) = (S2 (x) S1) vec(P)): with the input
// reshaped column-major, a SLAB = all (i_1, i_2) for one outer index
// J = (i_3..i_N) is S = d_1 d_2 contiguous floats, and it adds into ONE block of
// M12 = m_1 m_2 consecutive bins, at block g(J) = sum_{k>=3} h_k(i_k) prod_{3<=t<k} m_t,
// with the slab-internal map (h_1(i_1) + m_1 h_2(i_2), s_1 s_2) identical for every
// slab and the slab sign s(J) = prod_{k>=3} s_k(i_k).  A block of M12 bins holds
// M12/K whole tables, so the slabs of one block complete those tables.
//
// B200 mapping: persistent CTAs of 16 warps own tiles of 32 points (lane = point).
// The slabs of a tile are visited block by block; each slab is loaded (128-bit,
// two slabs in flight in registers), staged in shared memory in the slab's
// bin-sorted order with both signs applied (word pos*33 + lane: conflict-free
// stores and gathers), and every warp adds its M12/16 bins into registers.  After
// a block's last slab the codes are discretised and the block's tables keyed.
// Empty blocks (no slab maps there) still produce their keys (codes floor(b/w)).
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.hpp"

namespace lshb {

namespace {
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ uint64_t fmix64_h(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ int32_t floor_code_h(float q, int* flags) {
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
// a + sum of the C staged words listed at wo[0..C) (lane-relative base p)
template <int C>
__device__ __forceinline__ float sum_run(float a, const float* p, const uint16_t* wo) {
    float b = 0.f;   // two chains for ILP
#pragma unroll
    for (int c = 0; c < C; ++c) {
        if (c & 1) b += p[wo[c]];
        else a += p[wo[c]];
    }
    return a + b;
}
// The count of a (warp, bin) pair is the same for every slab of the kernel, so this
// switch always takes the same branch for a warp (no divergence, predictable).
__device__ __forceinline__ float sum_bin(float a, const float* p, const uint16_t* wo, uint32_t cnt) {
    switch (cnt) {
        case 0: return a;
        case 1: return sum_run<1>(a, p, wo);
        case 2: return sum_run<2>(a, p, wo);
        case 3: return sum_run<3>(a, p, wo);
        case 4: return sum_run<4>(a, p, wo);
        case 5: return sum_run<5>(a, p, wo);
        case 6: return sum_run<6>(a, p, wo);
        case 7: return sum_run<7>(a, p, wo);
        case 8: return sum_run<8>(a, p, wo);
        case 9: return sum_run<9>(a, p, wo);
        case 10: return sum_run<10>(a, p, wo);
        case 11: return sum_run<11>(a, p, wo);
        case 12: return sum_run<12>(a, p, wo);
        default:
            a = sum_run<12>(a, p, wo);
            for (uint32_t c = 12; c < cnt; ++c) a += p[wo[c]];
            return a;
    }
}
__device__ __forceinline__ float4 ldg_stream_h(const float* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
}  // namespace

// staged slab: word (k>>2)*129 + (k&3)*32 + r for coordinate k of row r (conflict-free
// for the staging stores of lane = column threads and for the lane = row gathers)
__host__ __device__ constexpr int hcs_tw(int S) { return (S / 4) * 129; }
constexpr int kHcsStep = 4;   // slab entries per step (one batch of loads, two barriers)

size_t hcs_smem_bytes(int S, int M12, int m, int ne, int nst) {
    (void)nst;
    return (size_t)kHcsStep * hcs_tw(S) * 4 + (size_t)S * 2 + (size_t)2 * M12 * 32 * 4 + (size_t)m * 4 +
           (size_t)ne * 8 + 64;
}

// CPW = S / 16, BPW = M12 / 16 (bins per warp)
template <int CPW, int BPW, bool E2>
__global__ void __launch_bounds__(kThreads, 1)
    sketch_hcs_kernel(HcsPlanDev plan, DiscretizeDev dz, const float* __restrict__ X, int64_t n, int64_t ld,
                      HashOut out, int dbg, int unused) {
    (void)unused;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int S = CPW * kWarps;
    constexpr int M12 = BPW * kWarps;
    constexpr int TW = hcs_tw(S);
    constexpr int Q4 = S / 4;              // float4 columns of a slab row
    constexpr int RPI = kThreads / Q4;     // rows per load iteration
    constexpr int VPT = 32 / RPI;          // float4 per thread per slab
    constexpr int NB = kHcsStep * VPT;     // float4 per thread per step
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m = plan.m, K = plan.K, ne = plan.nentries;   // ne: multiple of kHcsStep
    float* T = reinterpret_cast<float*>(smem_raw);                            // [kHcsStep][TW]
    uint16_t* wo = reinterpret_cast<uint16_t*>(T + kHcsStep * TW);            // [S]
    uint32_t* zs0 = reinterpret_cast<uint32_t*>(wo + S);                      // [2][M12][32]
    float* s_coff = reinterpret_cast<float*>(zs0 + 2 * M12 * 32);             // [m]
    uint2* ents = reinterpret_cast<uint2*>(s_coff + m);                       // [ne]
    const int64_t ntiles = (n + 31) >> 5;
    int64_t tile = blockIdx.x;
    if (tile >= ntiles) return;
    for (int i = tid; i < m; i += kThreads) s_coff[i] = E2 ? __ldg(dz.c_off + i) : 0.f;
    for (int i = tid; i < ne; i += kThreads) ents[i] = __ldg(plan.entries + i);
    for (int i = tid; i < S; i += kThreads) wo[i] = __ldg(plan.pos + i);
    __syncthreads();

    // staging column of this thread: coordinates 4*c4..4*c4+3 of rows r0 + v*RPI
    const int c4 = tid % Q4, r0 = tid / Q4;
    const uint32_t sg12 = (__ldg(plan.sgn + ((4 * c4) >> 5)) >> ((4 * c4) & 31)) & 0xfu;
    // this warp's bins (balanced by coordinate count at plan time): id, start, count
    uint32_t wb[BPW], bs[BPW], bc[BPW];
#pragma unroll
    for (int j = 0; j < BPW; ++j) {
        wb[j] = __ldg(plan.wbins + warp * BPW + j);
        bs[j] = __ldg(plan.bp + wb[j]);
        bc[j] = __ldg(plan.bp + wb[j] + 1) - bs[j];
    }
    int zpar = 0;

    float4 buf[NB];
    auto load = [&](int64_t tl, int e0) {
        const int64_t row0 = tl * 32 + r0;
#pragma unroll
        for (int q = 0; q < kHcsStep; ++q) {
            const uint2 ent = ents[e0 + q];
            const float* src = X + row0 * ld + (int64_t)ent.x * S + 4 * c4;
            const bool on = !(ent.y & HCS_EMPTY);
#pragma unroll
            for (int v = 0; v < VPT; ++v)
                buf[q * VPT + v] = (on && row0 + v * RPI < n) ? ldg_stream_h(src + (int64_t)v * RPI * ld)
                                                              : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    auto store = [&](int e0) {
#pragma unroll
        for (int q = 0; q < kHcsStep; ++q) {
            const uint2 ent = ents[e0 + q];
            const uint32_t sg = sg12 ^ ((ent.y & HCS_NEG) ? 0xfu : 0u);
            float* dst = T + q * TW + c4 * 129 + r0;
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                const float4 x = buf[q * VPT + v];
                dst[v * RPI] = __uint_as_float(__float_as_uint(x.x) ^ ((sg & 1u) << 31));
                dst[v * RPI + 32] = __uint_as_float(__float_as_uint(x.y) ^ (((sg >> 1) & 1u) << 31));
                dst[v * RPI + 64] = __uint_as_float(__float_as_uint(x.z) ^ (((sg >> 2) & 1u) << 31));
                dst[v * RPI + 96] = __uint_as_float(__float_as_uint(x.w) ^ (((sg >> 3) & 1u) << 31));
            }
        }
    };

    float acc[BPW];
#pragma unroll
    for (int j = 0; j < BPW; ++j) acc[j] = 0.f;
    const float cs = dz.c_scale;
    int e0 = 0;
    load(tile, e0);
    while (true) {
        __syncthreads();  // previous gathers done with T
        store(e0);
        __syncthreads();
        // next step's loads are in flight during the gathers below
        int64_t ntile = tile;
        int ne0 = e0 + kHcsStep;
        if (ne0 == ne) {
            ne0 = 0;
            ntile += gridDim.x;
        }
        const bool has_next = ntile < ntiles;
        if (has_next) load(ntile, ne0);
        const int64_t row = tile * 32 + lane;
        const bool valid = row < n;
#pragma unroll 1
        for (int q = 0; q < kHcsStep; ++q) {
            const uint2 ent = ents[e0 + q];
            if (!(ent.y & HCS_EMPTY)) {
                const float* p = T + q * TW + lane;
#pragma unroll
                for (int j = 0; j < BPW; ++j) acc[j] = sum_bin(acc[j], p, wo + bs[j], bc[j]);
            }
            if (ent.y & HCS_LAST) {
                const int g = (int)(ent.y & HCS_BLOCK_MASK);
                uint32_t* zs = zs0 + zpar * M12 * 32;   // double-buffered: no barrier after the keys
                zpar ^= 1;
#pragma unroll
                for (int j = 0; j < BPW; ++j) {
                    const int b = (int)wb[j];
                    const int l = g * M12 + b;
                    uint32_t z;
                    if constexpr (E2) {
                        z = (uint32_t)floor_code_h(fmaf(acc[j], cs, s_coff[l]), dz.flags);
                        if (dbg && valid && out.codes) out.codes[row * m + l] = (int32_t)z;
                    } else {
                        z = acc[j] > 0.0f ? 1u : 0u;
                        if (dbg && valid && out.bits && z)
                            atomicOr(&out.bits[row * ((m + 31) >> 5) + (l >> 5)], 1u << (l & 31));
                    }
                    if (dbg && valid && out.proj) out.proj[row * m + l] = acc[j];
                    zs[b * 32 + lane] = z;
                    acc[j] = 0.f;
                }
                __syncthreads();
                const int tpb = M12 / K;  // tables per block
                if (tid < tpb * 32) {
                    const int tb = tid >> 5;
                    uint64_t fp = E2 ? LSHB_FNV_OFFSET : 0ull;
                    for (int kk = 0; kk < K; ++kk) {
                        const uint32_t z = zs[(tb * K + kk) * 32 + lane];
                        if constexpr (E2) fp = (fp ^ (uint64_t)z) * LSHB_FNV_PRIME;
                        else fp |= (uint64_t)z << kk;
                    }
                    if (valid && out.keys) out.keys[(int64_t)(g * tpb + tb) * n + row] = E2 ? fmix64_h(fp) : fp;
                }
            }
        }
        if (!has_next) break;
        tile = ntile;
        e0 = ne0;
    }
}

template <int CPW, int BPW>
static cudaError_t launch_h(const HcsPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n, int64_t ld,
                            HashOut out, int num_sms, cudaStream_t s) {
    const int nst = 0;
    const size_t smem = hcs_smem_bytes(CPW * kWarps, BPW * kWarps, plan.m, plan.nentries, nst);
    const int64_t ntiles = (n + 31) / 32;
    const int grid = (int)(ntiles < num_sms ? ntiles : num_sms);
    const int dbg = (out.codes || out.bits || out.proj) ? 1 : 0;
    cudaError_t e;
    if (dz.e2lsh) {
        e = cudaFuncSetAttribute(sketch_hcs_kernel<CPW, BPW, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        if (e != cudaSuccess) return e;
        sketch_hcs_kernel<CPW, BPW, true><<<grid, kThreads, smem, s>>>(plan, dz, X, n, ld, out, dbg, nst);
    } else {
        e = cudaFuncSetAttribute(sketch_hcs_kernel<CPW, BPW, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        if (e != cudaSuccess) return e;
        sketch_hcs_kernel<CPW, BPW, false><<<grid, kThreads, smem, s>>>(plan, dz, X, n, ld, out, dbg, nst);
    }
    return cudaGetLastError();
}

bool hcs_plan_supported(int S, int M12) {
    return (S == 64 || S == 128 || S == 256) && (M12 == 16 || M12 == 32 || M12 == 64 || M12 == 128);
}

cudaError_t launch_sketch_hcs(const HcsPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n, int64_t ld,
                              HashOut out, int num_sms, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int cpw = plan.S / kWarps, bpw = plan.M12 / kWarps;
#define LSHB_HCS_CASE(C, B) \
    if (cpw == C && bpw == B) return launch_h<C, B>(plan, dz, X, n, ld, out, num_sms, s);
    LSHB_HCS_CASE(16, 4)
    LSHB_HCS_CASE(16, 2)
    LSHB_HCS_CASE(16, 8)
    LSHB_HCS_CASE(16, 1)
    LSHB_HCS_CASE(8, 4)
    LSHB_HCS_CASE(8, 2)
    LSHB_HCS_CASE(8, 1)
    LSHB_HCS_CASE(8, 8)
    LSHB_HCS_CASE(4, 4)
    LSHB_HCS_CASE(4, 2)
    LSHB_HCS_CASE(4, 1)
    LSHB_HCS_CASE(4, 8)
#undef LSHB_HCS_CASE
    return cudaErrorInvalidValue;
}

}  // namespace lshb
