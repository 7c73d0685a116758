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
#include <cuda.h>
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

// ---------------------------------------------------------------------------
// TMA variant (the default when X allows it): the same per-entry computation, but the
// slabs arrive by TMA — one cp.async.bulk.tensor.2d per (tile, slab), a 32-row x S
// box of X with out-of-range rows zero-filled — into an NS-stage shared ring issued by
// a producer warp, so no register holds in-flight data and more of it is in flight
// (NS x 32 KB per SM at S = 256 vs four 32 KB register buffers).  The 16 compute warps
// read their float4 columns of each slab from shared memory (conflict-free: a warp
// reads 512 contiguous bytes of a row), release the stage, and finalise blocks exactly
// as above (named barrier 1 over the 512 compute threads).
// ---------------------------------------------------------------------------
namespace {
__device__ __forceinline__ uint32_t hsm(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void hbar() { asm volatile("bar.sync 1, 512;" ::: "memory"); }
__device__ __forceinline__ void hm_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(hsm(b)), "r"(c));
}
__device__ __forceinline__ void hm_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(hsm(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void hm_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(hsm(b)) : "memory");
}
__device__ __forceinline__ void hm_wait(uint64_t* b, uint32_t ph) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LAB_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra LAB_WAIT_%=;\n"
        "}\n" ::"r"(hsm(b)),
        "r"(ph)
        : "memory");
}
__device__ __forceinline__ void h_tma2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            hsm(dst)),
        "l"(map), "r"(hsm(bar)), "r"(x), "r"(y)
        : "memory");
}
}  // namespace

constexpr int kHcsTmaThreads = kThreads + 32;
// shared memory of the TMA variant: T, wo, zs, entries, then NS stages (1 KB aligned) + barriers
__host__ __device__ inline size_t hcs_tma_fixed_bytes(int S, int M12, int ne) {
    size_t x = (size_t)hcs_tw(S) * 4 + (size_t)S * 2 + (size_t)2 * M12 * 32 * 4 + (size_t)ne * 8;
    return (x + 1023) / 1024 * 1024;
}
static size_t hcs_tma_smem(int S, int M12, int ne, int ns) {
    return hcs_tma_fixed_bytes(S, M12, ne) + (size_t)ns * 32 * S * 4 + (size_t)ns * 16 + 1024;
}

template <int CPW, int BPW, bool E2>
__global__ void __launch_bounds__(kHcsTmaThreads, 1)
    sketch_hcs_tma_kernel(const __grid_constant__ CUtensorMap xmap, HcsPlanDev plan, DiscretizeDev dz, int64_t n,
                          HashOut out, int dbg, int ns) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    constexpr int S = CPW * kWarps;
    constexpr int M12 = BPW * kWarps;
    constexpr int TW = hcs_tw(S);
    constexpr int Q4 = S / 4;
    constexpr int RPI = kThreads / Q4;
    constexpr int VPT = 32 / RPI;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m = plan.m, K = plan.K, ne = plan.nentries;
    // 1 KB-align the dynamic window (TMA destinations)
    unsigned char* base = smem_raw + ((1024 - (hsm(smem_raw) & 1023)) & 1023);
    float* T = reinterpret_cast<float*>(base);                                 // [TW]
    uint16_t* wo = reinterpret_cast<uint16_t*>(T + TW);                        // [S]
    uint32_t* zs0 = reinterpret_cast<uint32_t*>(wo + S);                       // [2][M12][32]
    uint2* ents = reinterpret_cast<uint2*>(zs0 + 2 * M12 * 32);                // [ne]
    float* stg = reinterpret_cast<float*>(base + hcs_tma_fixed_bytes(S, M12, ne));   // [ns][32][S]
    uint64_t* full = reinterpret_cast<uint64_t*>(stg + (size_t)ns * 32 * S);
    uint64_t* empty = full + ns;
    const int64_t ntiles = (n + 31) >> 5;
    if ((int64_t)blockIdx.x >= ntiles) return;
    for (int i = tid; i < ne; i += kHcsTmaThreads) ents[i] = __ldg(plan.entries + i);
    for (int i = tid; i < S; i += kHcsTmaThreads) wo[i] = __ldg(plan.pos + i);
    if (tid == kThreads) {
        for (int j = 0; j < ns; ++j) {
            hm_init(&full[j], 1u);
            hm_init(&empty[j], (uint32_t)kWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
    }
    __syncthreads();
    if (warp == kWarps) {
        // producer: every non-empty entry of every tile of this CTA, in consumption order
        if (lane == 0) {
            int sl = 0;
            uint32_t ph = 0;
            for (int64_t lt = blockIdx.x; lt < ntiles; lt += gridDim.x)
                for (int le = 0; le < ne; ++le) {
                    const uint2 ent = ents[le];
                    if (ent.y & HCS_EMPTY) continue;
                    hm_wait(&empty[sl], ph ^ 1u);
                    hm_expect(&full[sl], 32u * S * 4u);
                    h_tma2d(stg + (size_t)sl * 32 * S, &xmap, &full[sl], (int)(ent.x * S), (int)(lt * 32));
                    if (++sl == ns) {
                        sl = 0;
                        ph ^= 1u;
                    }
                }
        }
        return;
    }

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
    float4 z[VPT];
#pragma unroll
    for (int v = 0; v < VPT; ++v) z[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    const float cs = dz.c_scale;
    int zpar = 0, sl = 0;
    uint32_t ph = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t row = tile * 32 + lane;
        const bool valid = row < n;
        for (int ce = 0; ce < ne; ++ce) {
            const uint2 ent = ents[ce];
            if (!(ent.y & HCS_EMPTY)) {
                const float sgn = (ent.y & HCS_NEG) ? -1.f : 1.f;
                hm_wait(&full[sl], ph);
                const float* sp = stg + (size_t)sl * 32 * S + 4 * c4;
#pragma unroll
                for (int v = 0; v < VPT; ++v) {
                    const float4 b = *reinterpret_cast<const float4*>(sp + (size_t)(r0 + v * RPI) * S);
                    z[v].x = fmaf(sgn, b.x, z[v].x);
                    z[v].y = fmaf(sgn, b.y, z[v].y);
                    z[v].z = fmaf(sgn, b.z, z[v].z);
                    z[v].w = fmaf(sgn, b.w, z[v].w);
                }
                __syncwarp();
                if (lane == 0) hm_arrive(&empty[sl]);
                if (++sl == ns) {
                    sl = 0;
                    ph ^= 1u;
                }
            }
            if (!(ent.y & HCS_LAST)) continue;
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
            hbar();
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
                    zc = (uint32_t)floor_code(fmaf(y, cs, __ldg(dz.c_off + l)), dz.flags);
                    if (dbg && valid && out.codes) out.codes[row * m + l] = (int32_t)zc;
                } else {
                    zc = y > 0.0f ? 1u : 0u;
                    if (dbg && valid && out.bits && zc)
                        atomicOr(&out.bits[row * ((m + 31) >> 5) + (l >> 5)], 1u << (l & 31));
                }
                if (dbg && valid && out.proj) out.proj[row * m + l] = y;
                zs[b * 32 + lane] = zc;
            }
            hbar();   // codes complete; every gather is done with T
            const int tpb = M12 / K;  // tables per block
            if (tid < tpb * 32) {
                const int tb = tid >> 5;
                uint64_t fp = 0;
                FpKey fk;
                if (K == 16) {
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
                if (valid && out.keys && LSHB_OK(row < n))
                    out.keys[(int64_t)(g * tpb + tb) * n + row] = E2 ? fk.key() : fp;
            }
        }
    }
}

typedef CUresult (*PFN_hcsEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_hcsEncodeTiled hcs_encode() {
    static PFN_hcsEncodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_hcsEncodeTiled>(p);
    }
    return fn;
}

// TMA launch; returns cudaErrorNotSupported when X does not allow a tensor map (the
// caller then uses the register-fed kernel).
template <int CPW, int BPW>
static cudaError_t launch_h_tma(const HcsPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n, int64_t ld,
                                int64_t d, HashOut out, int num_sms, cudaStream_t s) {
    constexpr int S = CPW * kWarps;
    static const bool off = getenv("LSH_HCS_NO_TMA") && getenv("LSH_HCS_NO_TMA")[0] == '1';
    if (off || (reinterpret_cast<uintptr_t>(X) & 15) || (ld % 4) || n > 0x7fffffffll) return cudaErrorNotSupported;
    PFN_hcsEncodeTiled enc = hcs_encode();
    if (!enc) return cudaErrorNotSupported;
    // the slab columns [J*S, J*S+S) must lie inside the row: the slab plan only exists
    // when d is the product of the modes (no padding), so every J*S + S <= d
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {(cuuint32_t)S, 32u};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorNotSupported;
    int ns = 6;
    while (ns > 2 && hcs_tma_smem(S, BPW * kWarps, plan.nentries, ns) > 227 * 1024) --ns;
    const size_t smem = hcs_tma_smem(S, BPW * kWarps, plan.nentries, ns);
    if (smem > 227 * 1024) return cudaErrorNotSupported;
    const int64_t ntiles = (n + 31) / 32;
    const int grid = (int)(ntiles < num_sms ? ntiles : num_sms);
    const int dbg = (out.codes || out.bits || out.proj) ? 1 : 0;
    cudaError_t e;
    if (dz.e2lsh) {
        e = cudaFuncSetAttribute(sketch_hcs_tma_kernel<CPW, BPW, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        if (e != cudaSuccess) return e;
        sketch_hcs_tma_kernel<CPW, BPW, true><<<grid, kHcsTmaThreads, smem, s>>>(map, plan, dz, n, out, dbg, ns);
    } else {
        e = cudaFuncSetAttribute(sketch_hcs_tma_kernel<CPW, BPW, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        if (e != cudaSuccess) return e;
        sketch_hcs_tma_kernel<CPW, BPW, false><<<grid, kHcsTmaThreads, smem, s>>>(map, plan, dz, n, out, dbg, ns);
    }
    return cudaGetLastError();
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
#define LSHB_HCS_CASE(C, B)                                                                 \
    if (cpw == C && bpw == B) {                                                              \
        const cudaError_t et = launch_h_tma<C, B>(plan, dz, X, n, ld, plan.d, out, num_sms, s); \
        if (et != cudaErrorNotSupported) return et;                                          \
        return launch_h<C, B>(plan, dz, X, n, ld, out, num_sms, s);                          \
    }
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
