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

#include "discretize.cuh"
#include "internal.hpp"

namespace lshb {

namespace {
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;

// a + sum of the cnt staged words listed at wo[0..cnt) (lane-relative base p); two
// independent chains, the second half of each pair predicated
__device__ __forceinline__ float sum_bin(float a, const float* p, const uint16_t* wo, uint32_t cnt) {
    float b = 0.f;
    uint32_t c = 0;
#pragma unroll 2
    for (; c + 1 < cnt; c += 2) {
        a += p[wo[c]];
        b += p[wo[c + 1]];
    }
    if (c < cnt) a += p[wo[c]];
    return a + b;
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
// shared memory: the staged block sum, the bin-sorted coordinate list, block codes
// (double-buffered), b/w, entries
size_t hcs_smem_bytes(int S, int M12, int m, int ne, int nst) {
    (void)nst;
    return (size_t)hcs_tw(S) * 4 + (size_t)S * 2 + (size_t)2 * M12 * 32 * 4 + (size_t)m * 4 + (size_t)ne * 8 + 64;
}


// CPW = S / 16, BPW = M12 / 16 (bins per warp).
//
// Block sums first: all slabs J of block g share the slab-internal map, so
//   y_{g,b} = sum_J s(J) sum_{k in b} s12(k) x_J[k] = sum_{k in b} s12(k) Z_g[k],
//   Z_g = sum_J s(J) x_J   (element-wise).
// Z_g accumulates in registers (lane = column: one FFMA per input, no shared
// memory); the slab map is applied once per block.  Each thread streams its own
// 16-byte columns of every slab with 128-bit no-allocate loads into four rotating
// register buffers (four slabs, 128 KB per SM, in flight), so the streaming loop
// needs no block barrier; two barriers per block (stage Z_g transposed, then
// gather bins / key the block's tables).
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
    constexpr int RPI = kThreads / Q4;     // rows per thread step
    constexpr int VPT = 32 / RPI;          // float4 per thread per slab
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m = plan.m, K = plan.K, ne = plan.nentries;
    float* T = reinterpret_cast<float*>(smem_raw);                            // [TW]
    uint16_t* wo = reinterpret_cast<uint16_t*>(T + TW);                       // [S]
    uint32_t* zs0 = reinterpret_cast<uint32_t*>(wo + S);                      // [2][M12][32]
    float* s_coff = reinterpret_cast<float*>(zs0 + 2 * M12 * 32);             // [m]
    uint2* ents = reinterpret_cast<uint2*>(s_coff + m);                       // [ne]
    const int64_t ntiles = (n + 31) >> 5;
    if ((int64_t)blockIdx.x >= ntiles) return;
    for (int i = tid; i < m; i += kThreads) s_coff[i] = E2 ? __ldg(dz.c_off + i) : 0.f;
    for (int i = tid; i < ne; i += kThreads) ents[i] = __ldg(plan.entries + i);
    for (int i = tid; i < S; i += kThreads) wo[i] = __ldg(plan.pos + i);
    __syncthreads();

    const int c4 = tid % Q4, r0 = tid / Q4;
    const uint32_t sg12 = (__ldg(plan.sgn + ((4 * c4) >> 5)) >> ((4 * c4) & 31)) & 0xfu;
    const uint32_t sgm0 = (sg12 & 1u) << 31, sgm1 = ((sg12 >> 1) & 1u) << 31, sgm2 = ((sg12 >> 2) & 1u) << 31,
                   sgm3 = ((sg12 >> 3) & 1u) << 31;
    uint32_t wb[BPW], bs[BPW], bc[BPW];
#pragma unroll
    for (int j = 0; j < BPW; ++j) {
        wb[j] = __ldg(plan.wbins + warp * BPW + j);
        bs[j] = __ldg(plan.bp + wb[j]);
        bc[j] = __ldg(plan.bp + wb[j] + 1) - bs[j];
    }
    const int64_t vstride = (int64_t)RPI * ld;

    // (tile, entry) cursors advanced incrementally (no 64-bit division per entry):
    // `ct, ce` = entry being consumed, `lt, le` = entry being loaded (four ahead)
    int64_t lt = blockIdx.x;
    int le = 0;
    auto load = [&](float4* buf) {   // loads entry (lt, le), then advances the cursor
        if (lt < ntiles) {
            const uint2 ent = ents[le];
            if (!(ent.y & HCS_EMPTY)) {
                const int64_t row0 = lt * 32 + r0;
                const float* src = X + row0 * ld + (int64_t)ent.x * S + 4 * c4;
                if (lt * 32 + 32 <= n) {
#pragma unroll
                    for (int v = 0; v < VPT; ++v) buf[v] = ldg_stream_h(src + v * vstride);
                } else {
#pragma unroll
                    for (int v = 0; v < VPT; ++v)
                        buf[v] = row0 + v * RPI < n ? ldg_stream_h(src + v * vstride) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        }
        if (++le == ne) {
            le = 0;
            lt += gridDim.x;
        }
    };
    float4 bA[VPT], bB[VPT], bC[VPT], bD[VPT];
    load(bA);
    load(bB);
    load(bC);
    load(bD);

    float4 z[VPT];
#pragma unroll
    for (int v = 0; v < VPT; ++v) z[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    const float cs = dz.c_scale;
    int zpar = 0;
    int64_t tile = blockIdx.x;
    int ce = 0;
    // one entry: fold its slab (from `buf`) into Z, refill `buf` with the entry four
    // ahead, and after a block's last slab turn Z into the block's codes and keys
    auto step = [&](float4* buf) -> bool {
        if (tile >= ntiles) return true;
        const uint2 ent = ents[ce];
        if (!(ent.y & HCS_EMPTY)) {
            const float sgn = (ent.y & HCS_NEG) ? -1.f : 1.f;
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                z[v].x = fmaf(sgn, buf[v].x, z[v].x);
                z[v].y = fmaf(sgn, buf[v].y, z[v].y);
                z[v].z = fmaf(sgn, buf[v].z, z[v].z);
                z[v].w = fmaf(sgn, buf[v].w, z[v].w);
            }
        }
        load(buf);
        const int64_t row = tile * 32 + lane;
        if (++ce == ne) {
            ce = 0;
            tile += gridDim.x;
        }
        if (!(ent.y & HCS_LAST)) return false;
        // ---- block complete: stage Z_g (transposed, slab-internal sign applied) ----
        {
            float* dst = T + c4 * 129 + r0;
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                dst[v * RPI] = __uint_as_float(__float_as_uint(z[v].x) ^ sgm0);
                dst[v * RPI + 32] = __uint_as_float(__float_as_uint(z[v].y) ^ sgm1);
                dst[v * RPI + 64] = __uint_as_float(__float_as_uint(z[v].z) ^ sgm2);
                dst[v * RPI + 96] = __uint_as_float(__float_as_uint(z[v].w) ^ sgm3);
                z[v] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        __syncthreads();
        const bool valid = row < n;
        const int g = (int)(ent.y & HCS_BLOCK_MASK);
        uint32_t* zs = zs0 + zpar * M12 * 32;   // double-buffered: no barrier after the keys
        zpar ^= 1;
        const float* p = T + lane;
#pragma unroll
        for (int j = 0; j < BPW; ++j) {
            const float y = bc[j] ? sum_bin(0.f, p, wo + bs[j], bc[j]) : 0.f;
            const int b = (int)wb[j];
            const int l = g * M12 + b;
            uint32_t zc;
            if constexpr (E2) {
                zc = (uint32_t)floor_code(fmaf(y, cs, s_coff[l]), dz.flags);
                if (dbg && valid && out.codes) out.codes[row * m + l] = (int32_t)zc;
            } else {
                zc = y > 0.0f ? 1u : 0u;
                if (dbg && valid && out.bits && zc) atomicOr(&out.bits[row * ((m + 31) >> 5) + (l >> 5)], 1u << (l & 31));
            }
            if (dbg && valid && out.proj) out.proj[row * m + l] = y;
            zs[b * 32 + lane] = zc;
        }
        __syncthreads();   // codes complete; every gather is done with T
        const int tpb = M12 / K;  // tables per block
        if (tid < tpb * 32) {
            const int tb = tid >> 5;
            uint64_t fp = 0;
            FpKey fk;
            if (K == 16) {   // the usual K: all 16 codes loaded at once, the chain back to back
                uint32_t zk[16];
#pragma unroll
                for (int kk = 0; kk < 16; ++kk) zk[kk] = zs[(tb * 16 + kk) * 32 + lane];
#pragma unroll
                for (int kk = 0; kk < 16; ++kk) {
                    if constexpr (E2) fk.add(zk[kk]);
                    else fp |= (uint64_t)zk[kk] << kk;
                }
            } else {
                for (int kk = 0; kk < K; ++kk) {
                    const uint32_t zc = zs[(tb * K + kk) * 32 + lane];
                    if constexpr (E2) fk.add(zc);
                    else fp |= (uint64_t)zc << kk;
                }
            }
            if (valid && out.keys && LSHB_OK(row < n)) out.keys[(int64_t)(g * tpb + tb) * n + row] = E2 ? fk.key() : fp;
        }
        return false;
    };
    while (true) {
        if (step(bA)) break;
        if (step(bB)) break;
        if (step(bC)) break;
        if (step(bD)) break;
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
