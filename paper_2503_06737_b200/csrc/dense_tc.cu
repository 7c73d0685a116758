// dense_tc.cu — K4: the dense O(md) E2LSH / SRP projection Y = X R^T
// (PAPER.md:169 eq:datar_lsh, :187 Def. SRP; Table 1) on the 5th
// generation tensor cores (tcgen05.mma, accumulators in TMEM, operands staged by
// TMA with 128-byte swizzle).
//
// Exactness (reading B13): R is bf16-exact by construction, and each fp32
// input is split into three bf16 terms x = x0 + x1 + x2 (exact for normal values),
// so Y = [x0|x1|x2] . [R|R|R]^T is ONE bf16 GEMM over K' = 3*d_pad with fp32
// accumulation: every product is exact, only the fp32 accumulation rounds.
//
// Kernel shape (persistent, one CTA per SM walking output tiles, warp-specialised,
// 576 threads; two TMEM accumulator buffers so a tile's epilogue overlaps the
// next tile's MMAs):
//   warp 0      TMA producer: A tile 128 x 64 and B tile BN x 64 (bf16, SW128) per stage
//   warp 1      TMEM allocation + MMA issue (one elected thread, UMMA 128 x BN x 16)
//   warps 2..17 epilogue: tcgen05.ld 32 lanes x 16 columns at a time -> Y (fp32), or
//               (fused, KT > 0) the discretisation + table keys straight from TMEM:
//               16/KT whole tables per load, only the keys [L][n] reach HBM
//               (codes as the sketches compute them, discretize.cuh)
// 4-stage smem ring with full/empty mbarriers; tcgen05.commit frees a stage and
// finally signals the epilogue.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "discretize.cuh"
#include "internal.hpp"

namespace lshb {

namespace tc {
constexpr int BM = 128, BK = 64, STAGES = 4;
constexpr int EPI_WARPS = 16;                 // 4 per TMEM lane quadrant, each a quarter of the columns
constexpr int THREADS = 64 + 32 * EPI_WARPS;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LAB_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra LAB_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major operand tile written by TMA with 128-byte swizzle: rows of 128 B
// (64 bf16), 8-row swizzle atoms of 1024 B.  UMMA smem descriptor (sm100):
// start>>4 [0,14), LBO>>4 [16,30) (unused for swizzled K-major: 1), SBO>>4 [32,46)
// = 1024 B between 8-row groups, version 1 [46,48), layout SWIZZLE_128B = 2 [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// Instruction descriptor kind::f16: D fp32 (bit 4), A bf16 (bits 7-9 = 1), B bf16
// (bits 10-12 = 1), both K-major, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
}  // namespace tc

// Fused key epilogue (KT > 0): keys of table t for local row r at keys[t * kstride + r].
struct KeyEpi {
    uint64_t* keys;
    int64_t kstride;
    DiscretizeDev dz;
};

template <int BN, int KT>
__global__ void __launch_bounds__(tc::THREADS, 1)
    dense_tc_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b, int n,
                    int m, int d_pad, int nk, float* __restrict__ Y, KeyEpi ke) {
    using namespace tc;
    constexpr uint32_t A_BYTES = BM * BK * 2;   // 16 KB
    constexpr uint32_t B_BYTES = BN * BK * 2;
    constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
    // two accumulator buffers (the epilogue of tile i overlaps the MMAs of tile i+1)
    constexpr uint32_t ACC_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
    constexpr uint32_t TMEM_COLS = 2 * ACC_COLS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment of every operand tile (SW128 atoms)
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;    // [2] accumulator ready (MMA commit)
    uint64_t* tmem_empty = tmem_full + 2;    // [2] accumulator drained (one arrive per epilogue warp)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // persistent: tiles t = blockIdx.x + i * gridDim.x, column tiles fastest (the CTAs
    // in flight share A row tiles and walk B in step, so both stay L2-resident)
    const int ntn = (m + BN - 1) / BN;
    const int ntiles = ntn * ((n + BM - 1) / BM);

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_b) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // TMA producer: one k-block stream across all of this CTA's tiles
            uint32_t g = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int n_tile = tile % ntn, m_tile = tile / ntn;
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int s = g % STAGES;
                    const uint32_t ph = (g / STAGES) & 1;
                    mbar_wait(&empty[s], ph ^ 1);
                    unsigned char* a_dst = smem + s * STAGE_BYTES;
                    unsigned char* b_dst = a_dst + A_BYTES;
                    mbar_expect_tx(&full[s], STAGE_BYTES);
                    tma_load_2d(a_dst, &tmap_a, &full[s], kb * BK, m_tile * BM);
                    tma_load_2d(b_dst, &tmap_b, &full[s], (kb * BK) % d_pad, n_tile * BN);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // MMA issuer: UMMA_K = 16 (32 bytes of K per instruction)
            constexpr uint32_t idesc = idesc_bf16(BM, BN);
            uint32_t g = 0, i = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
                const uint32_t acc = i & 1;
                mbar_wait(&tmem_empty[acc], ((i >> 1) & 1) ^ 1);   // the epilogue drained this buffer
                fence_after();
                const uint32_t tmem_d = tmem_base + acc * ACC_COLS;
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int s = g % STAGES;
                    const uint32_t ph = (g / STAGES) & 1;
                    mbar_wait(&full[s], ph);
                    fence_after();
                    const uint32_t a_addr = smem_u32(smem + s * STAGE_BYTES);
                    const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        const uint64_t ad = sw128_desc(a_addr + k * 32);
                        const uint64_t bd = sw128_desc(b_addr + k * 32);
                        umma_bf16(tmem_d, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
                    }
                    umma_commit(&empty[s]);  // frees the stage when these MMAs complete
                }
                umma_commit(&tmem_full[acc]);   // accumulator ready
            }
        }
        __syncwarp();
    } else {
        // epilogue: warp w reads TMEM lanes [32*(w%4), +32) = tile rows
        const int q = warp & 3;                        // tcgen05.ld: lanes [32 (warp % 4), +32)
        const int slice = (warp - 2) >> 2;             // column slice of this warp in its quadrant
        uint32_t i = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
            const int n_tile = tile % ntn, m_tile = tile / ntn;
            const uint32_t acc = i & 1;
            mbar_wait(&tmem_full[acc], (i >> 1) & 1);
            fence_after();
            const int row = m_tile * BM + q * 32 + lane;
#pragma unroll 1
            for (int c0 = slice * 16; c0 < BN; c0 += 16 * (EPI_WARPS / 4)) {
                uint32_t v[16];
                const uint32_t taddr = tmem_base + acc * ACC_COLS + ((uint32_t)(q * 32) << 16) + (uint32_t)c0;
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                    "[%16];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const int col = n_tile * BN + c0;
                if constexpr (KT > 0) {
                    // 16 / KT tables: code l = col + j, table (col + j) / KT (tables never straddle)
#pragma unroll
                    for (int tb = 0; tb < 16 / KT; ++tb) {
                        const int l0 = col + tb * KT;
                        if (l0 >= m) break;
                        uint64_t f;
                        if (ke.dz.e2lsh) {
                            FpKey fk;
#pragma unroll
                            for (int kk = 0; kk < KT; ++kk) {
                                const float qv = fmaf(__uint_as_float(v[tb * KT + kk]), ke.dz.c_scale,
                                                      __ldg(ke.dz.c_off + l0 + kk));
                                fk.add((uint32_t)floor_code(qv, ke.dz.flags));
                            }
                            f = fk.key();
                        } else {
                            f = 0;
#pragma unroll
                            for (int kk = 0; kk < KT; ++kk)
                                f |= (__uint_as_float(v[tb * KT + kk]) > 0.0f ? 1ull : 0ull) << kk;
                        }
                        if (row < n) ke.keys[(int64_t)(l0 / KT) * ke.kstride + row] = f;
                    }
                    continue;
                }
                if (row < n) {
                    float* dst = Y + (int64_t)row * m + col;
                    if (col + 16 <= m && (m % 4) == 0) {
#pragma unroll
                        for (int j = 0; j < 16; j += 4)
                            *reinterpret_cast<float4*>(dst + j) =
                                make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                                            __uint_as_float(v[j + 3]));
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (col + j < m) dst[j] = __uint_as_float(v[j]);
                    }
                }
            }
            // this warp is done with the buffer: let the MMA warp overwrite it
            fence_before();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tmem_empty[acc])) : "memory");
        }
    }
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    }
}

// x (fp32) -> [x0 | x1 | x2] bf16, row length 3*d_pad, zero padded (exact split).
// Block per row (grid-stride over rows), thread per 4 consecutive columns: one
// 128-bit load (when rows are 16-byte aligned) and one 8-byte store per term.
__device__ __forceinline__ uint32_t pack_bf16x2(__nv_bfloat16 lo, __nv_bfloat16 hi) {
    return (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
}
__global__ void __launch_bounds__(256) split3_kernel(const float* __restrict__ X, int64_t n, int64_t ld, int d,
                                                     int d_pad, int vec_ok, __nv_bfloat16* __restrict__ A) {
    const int q4 = d_pad >> 2;
    for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
        const float* xr = X + r * ld;
        uint2* row = reinterpret_cast<uint2*>(A + r * (int64_t)(3 * d_pad));
        for (int c4 = threadIdx.x; c4 < q4; c4 += blockDim.x) {
            const int k = 4 * c4;
            float v[4];
            if (vec_ok && k + 4 <= d) {
                const float4 f = __ldcs(reinterpret_cast<const float4*>(xr + k));
                v[0] = f.x;
                v[1] = f.y;
                v[2] = f.z;
                v[3] = f.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) v[j] = k + j < d ? xr[k + j] : 0.f;
            }
            __nv_bfloat16 t0[4], t1[4], t2[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                t0[j] = __float2bfloat16_rn(v[j]);
                const float r1 = v[j] - __bfloat162float(t0[j]);
                t1[j] = __float2bfloat16_rn(r1);
                const float r2 = r1 - __bfloat162float(t1[j]);
                t2[j] = __float2bfloat16_rn(r2);
            }
            row[c4] = make_uint2(pack_bf16x2(t0[0], t0[1]), pack_bf16x2(t0[2], t0[3]));
            row[q4 + c4] = make_uint2(pack_bf16x2(t1[0], t1[1]), pack_bf16x2(t1[2], t1[3]));
            row[2 * q4 + c4] = make_uint2(pack_bf16x2(t2[0], t2[1]), pack_bf16x2(t2[2], t2[3]));
        }
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    }
    return fn;
}

static bool make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                     uint32_t box_inner, uint32_t box_outer) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t dense_tc_rows_per_batch(int d_pad) {
    // A' scratch = rows * 3 * d_pad * 2 bytes; cap at ~2 GB
    size_t rows = (size_t)2 << 30;
    rows /= (size_t)3 * d_pad * 2;
    rows = rows / 128 * 128;
    if (rows < 128) rows = 128;
    return rows;
}

template <int BN, int KT>
static cudaError_t launch_tc_k(const CUtensorMap& ma, const CUtensorMap& mb, int n, int m, int d_pad, float* Y,
                               const KeyEpi& ke, cudaStream_t s) {
    const size_t smem = (size_t)tc::STAGES * (tc::BM * tc::BK * 2 + BN * tc::BK * 2) + 1024 + 256;
    cudaError_t e =
        cudaFuncSetAttribute(dense_tc_kernel<BN, KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int nk = 3 * d_pad / tc::BK;
    const int ntiles = ((m + BN - 1) / BN) * ((n + tc::BM - 1) / tc::BM);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = ntiles < sms ? ntiles : sms;   // persistent: one CTA per SM
    dense_tc_kernel<BN, KT><<<grid, tc::THREADS, smem, s>>>(ma, mb, n, m, d_pad, nk, Y, ke);
    return cudaGetLastError();
}

template <int BN>
static cudaError_t launch_tc_t(const CUtensorMap& ma, const CUtensorMap& mb, int n, int m, int d_pad, float* Y,
                               const KeyEpi& ke, int K, cudaStream_t s) {
    if (!ke.keys) return launch_tc_k<BN, 0>(ma, mb, n, m, d_pad, Y, ke, s);
    switch (K) {
        case 16: return launch_tc_k<BN, 16>(ma, mb, n, m, d_pad, Y, ke, s);
        case 8: return launch_tc_k<BN, 8>(ma, mb, n, m, d_pad, Y, ke, s);
        case 4: return launch_tc_k<BN, 4>(ma, mb, n, m, d_pad, Y, ke, s);
        case 2: return launch_tc_k<BN, 2>(ma, mb, n, m, d_pad, Y, ke, s);
        case 1: return launch_tc_k<BN, 1>(ma, mb, n, m, d_pad, Y, ke, s);
    }
    return cudaErrorInvalidValue;
}

bool dense_tc_fused_keys_ok(int m, int K) {
    const int BN = m >= 256 ? 256 : (m > 128 ? ((m + 15) / 16) * 16 : 128);
    return K >= 1 && K <= 16 && (16 % K) == 0 && (BN % K) == 0 && (m % K) == 0;
}

// Y [n][m] = X R^T with R_pad bf16 [m][d_pad] (zero padded), A scratch bf16 [rows][3*d_pad].
// keys != nullptr: fused key epilogue (requires dense_tc_fused_keys_ok(m, K)), Y unused.
cudaError_t launch_dense_tc(const float* X, int64_t n, int64_t ld, int d, const uint16_t* R_pad, int m, int d_pad,
                            uint16_t* A_scratch, int64_t rows_per_batch, float* Y, cudaStream_t s, uint64_t* keys,
                            int K, const DiscretizeDev* dz) {
    if (n == 0) return cudaSuccess;
    CUtensorMap mb;
    const int BN = m >= 256 ? 256 : (m > 128 ? ((m + 15) / 16) * 16 : 128);
    if (!make_map(&mb, R_pad, (uint64_t)d_pad, (uint64_t)m, (uint64_t)d_pad * 2, tc::BK, (uint32_t)(BN > 256 ? 256 : BN)))
        return cudaErrorInvalidValue;
    for (int64_t r0 = 0; r0 < n; r0 += rows_per_batch) {
        const int64_t nb = n - r0 < rows_per_batch ? n - r0 : rows_per_batch;
        const int vec_ok = ((ld % 4) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0) ? 1 : 0;
        const int blocks = (int)(nb < 148 * 16 ? nb : 148 * 16);
        split3_kernel<<<blocks, 256, 0, s>>>(X + r0 * ld, nb, ld, d, d_pad, vec_ok,
                                             reinterpret_cast<__nv_bfloat16*>(A_scratch));
        count_launch();
        CUtensorMap ma;
        if (!make_map(&ma, A_scratch, (uint64_t)3 * d_pad, (uint64_t)nb, (uint64_t)3 * d_pad * 2, tc::BK, tc::BM))
            return cudaErrorInvalidValue;
        KeyEpi ke{};
        float* Yb = keys ? nullptr : Y + r0 * m;
        if (keys) {
            ke.keys = keys + r0;
            ke.kstride = n;
            ke.dz = *dz;
        }
        cudaError_t e;
        if (BN == 256) e = launch_tc_t<256>(ma, mb, (int)nb, m, d_pad, Yb, ke, K, s);
        else if (BN == 128) e = launch_tc_t<128>(ma, mb, (int)nb, m, d_pad, Yb, ke, K, s);
        else if (BN == 160) e = launch_tc_t<160>(ma, mb, (int)nb, m, d_pad, Yb, ke, K, s);
        else if (BN == 192) e = launch_tc_t<192>(ma, mb, (int)nb, m, d_pad, Yb, ke, K, s);
        else if (BN == 144) e = launch_tc_t<144>(ma, mb, (int)nb, m, d_pad, Yb, ke, K, s);
        else if (BN == 176) e = launch_tc_t<176>(ma, mb, (int)nb, m, d_pad, Yb, ke, K, s);
        else if (BN == 208) e = launch_tc_t<208>(ma, mb, (int)nb, m, d_pad, Yb, ke, K, s);
        else if (BN == 224) e = launch_tc_t<224>(ma, mb, (int)nb, m, d_pad, Yb, ke, K, s);
        else if (BN == 240) e = launch_tc_t<240>(ma, mb, (int)nb, m, d_pad, Yb, ke, K, s);
        else e = cudaErrorInvalidValue;
        count_launch();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace lshb
