// group.cu — K3/K5: grouping points into the buckets of each of the L tables
// ("store every point p in bucket hbar_t(p)"; "arranging data
// points into several bins of hash tables based on their hashcode")
// and the bucket lookup of queries.  DESIGN.md §K3.
//
// Output order is canonical (reading B11): per table, ids sorted by (key, id),
// i.e. buckets by ascending unsigned key, ids ascending inside a bucket.
//
// B200 design (two passes over the keys after the histogram):
//   L1  one stable MSD counting scatter of every table on its top B1 key bits
//       (B1 = 1..11 chosen so bins average <= 2048 items).  The destination of
//       one table (12 B x n) stays resident in the 126 MB L2 while the grid
//       works on that table, so the scattered runs merge in L2 before they
//       reach HBM.  Stability comes from warp-private match_any ranking.
//   L2  one CTA per (bin, table): the bin is loaded into shared memory and
//       sorted there by the next 16 key bits (two stable 8-bit passes on a
//       16-bit permutation), equal-prefix segments are finished by O(s) ranks
//       (long ones by further passes), then run-length encoded.  The bucket
//       numbering across bins is a decoupled look-back (chained) scan, so ids,
//       ukeys and offs are written once, compacted, in the same kernel.
//   Bins larger than shared memory (skewed codes: many equal keys) take the
//   same algorithm on global memory: a stable 3-way split around a dominant
//   key, then stable 8-bit passes over the varying digits only.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>

#include "internal.hpp"

namespace lshb {

#ifndef LSHB_G1_TILE
#define LSHB_G1_TILE 8192
#endif
#ifndef LSHB_SCATTER_CPS
#define LSHB_SCATTER_CPS 1   // L1 scatter CTAs per SM
#endif
constexpr int kG1Tile = LSHB_G1_TILE;           // items per L1 tile
constexpr int kG1Threads = 256;
constexpr int kG2Threads = 512;
constexpr int kG2Warps = kG2Threads / 32;       // 16
constexpr int kG2Cap = 4096;                    // run-length-encoding chunk (narrow keys)
#ifndef LSHB_G2_T
#define LSHB_G2_T 256    // threads of the per-bin sort CTA (g2a)
#endif
#ifndef LSHB_G2_IPT
#define LSHB_G2_IPT (1280 / LSHB_G2_T)   // items per thread of g2a: bin capacity T * IPT = 1280
#endif
#ifndef LSHB_G2_CPS
#define LSHB_G2_CPS (LSHB_G2_T == 128 ? 6 : 5)   // g2a CTAs per SM (launch bound)
#endif
#ifndef LSHB_G2_D
#define LSHB_G2_D 12     // counting-sort digit bits inside a bin
#endif
#ifndef LSHB_L1_AVG
#define LSHB_L1_AVG 1024 // L1 bins hold at most this many keys on average
#endif
constexpr int kG2BinCap = LSHB_G2_T * LSHB_G2_IPT;    // largest L1 bin sorted in shared memory (g2a)

size_t group_tiles(int64_t n) { return (size_t)((n + kG1Tile - 1) / kG1Tile); }

// Narrow keys (SRP codes, K <= 22) are sorted completely by two stable LSD passes
// over their varying bits (<= 11 each); wide keys (E2LSH fingerprints) by one MSD
// pass + the per-chunk shared-memory sort.
bool group_is_lsd(int W) { return W <= 22; }

int group_l1_bits(int64_t n, int W) {
    if (group_is_lsd(W)) return (W + 1) / 2;
    int b = 1;
    while (b < 11 && ((n + (1ll << b) - 1) >> b) > LSHB_L1_AVG) ++b;   // bins of <= LSHB_L1_AVG on average
    return b < W ? b : W;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// Lanes of the warp holding the same digit (digits < 2^NB; invalid lanes match only
// themselves): one ballot per digit bit instead of match.any, whose cost grows with
// the number of distinct values (about 32 here).
template <int NB>
__device__ __forceinline__ uint32_t match_digit(uint32_t d, int nbits, bool valid) {
    uint32_t m = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        if (b < nbits) {
            const bool bit = (d >> b) & 1u;
            const uint32_t bb = __ballot_sync(0xffffffffu, bit);
            m &= bit ? bb : ~bb;
        }
    }
    return valid ? m : (1u << (threadIdx.x & 31));
}

// Exclusive block scan of one value per thread (NT threads); optional total.
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* ws, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < NT / 32 ? ws[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NT / 32) ws[lane] = w;
    }
    __syncthreads();
    const uint32_t r = (warp ? ws[warp - 1] : 0u) + x - v;
    if (total) *total = ws[NT / 32 - 1];
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------------------
// L1 digit selection: the top B1 key bits that VARY over the table.  SRP keys
// have constant bits (sketch bins with no coordinate, sign patterns shared by a
// cluster), so a fixed top-bits digit would collapse into a few huge bins.
// Extracting varying bits keeps key order (the other bits are constant).
// ---------------------------------------------------------------------------
struct L1Spec {
    uint64_t below;   // key bits below the lowest digit bit: what the per-bin sort still orders
    int32_t nbits;    // digit bits (<= B1; fewer when fewer key bits vary)
    int32_t shift;    // contiguous digit: (key >> shift) & (2^nbits - 1); -1: gather pos[]
    uint8_t pos[12];  // digit bit positions, most significant first
};

__device__ __forceinline__ uint32_t l1_digit(uint64_t k, const L1Spec& s) {
    if (s.shift >= 0) return (uint32_t)(k >> s.shift) & ((1u << s.nbits) - 1u);
    uint32_t d = 0;
#pragma unroll
    for (int j = 0; j < 11; ++j)
        if (j < s.nbits) d = (d << 1) | (uint32_t)((k >> s.pos[j]) & 1ull);
    return d;
}

// OR of the keys and OR of their complements per table (varying bits = both set).
__global__ void __launch_bounds__(256) g0_mask(const uint64_t* __restrict__ keys, int64_t n,
                                               unsigned long long* __restrict__ vm) {
    const int t = blockIdx.y;
    const uint64_t* kt = keys + (int64_t)t * n;
    uint64_t o = 0, no = 0;
    const int64_t i0 = (int64_t)blockIdx.x * 8192 + threadIdx.x;
#pragma unroll 8
    for (int r = 0; r < 32; ++r) {
        const int64_t i = i0 + r * 256;
        if (i < n) {
            const uint64_t k = __ldcs(kt + i);
            o |= k;
            no |= ~k;
        }
    }
#pragma unroll
    for (int sft = 16; sft > 0; sft >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, sft);
        no |= __shfl_xor_sync(0xffffffffu, no, sft);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicOr(vm + 2 * t, (unsigned long long)o);
        atomicOr(vm + 2 * t + 1, (unsigned long long)no);
    }
}

__device__ L1Spec make_spec(const int* pos, int nb) {
    L1Spec s;
    s.nbits = nb;
    for (int j = 0; j < 12; ++j) s.pos[j] = j < nb ? (uint8_t)pos[j] : 0;
    if (nb == 0) {
        s.shift = 0;
        s.below = ~0ull;
    } else {
        const int lo = pos[nb - 1];
        s.shift = (pos[0] - lo == nb - 1) ? lo : -1;
        s.below = (1ull << lo) - 1ull;
    }
    return s;
}

// passes == 1 (MSD): the top B1 varying bits.  passes == 2 (LSD, narrow keys): the
// varying bits split into a low half (pass 0) and a high half (pass 1), each <= B1.
__global__ void g0_spec(const unsigned long long* __restrict__ vm, int L, int B1, int passes,
                        L1Spec* __restrict__ spec, const uint32_t* __restrict__ gate = nullptr) {
    if (gate && *gate == 0u) return;   // (gated: runs only as the fixed-capacity path's fallback)
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= L) return;
    const uint64_t V = vm[2 * t] & vm[2 * t + 1];
    int pos[64];
    int v = 0;
    for (int b = 63; b >= 0; --b)
        if ((V >> b) & 1ull) pos[v++] = b;
    if (passes == 1) {
        spec[t] = make_spec(pos, v < B1 ? v : B1);
    } else {
        const int hi_n = min(B1, (v + 1) / 2);
        const int lo_n = min(B1, v - hi_n);
        spec[(int64_t)L + t] = make_spec(pos, hi_n);   // pass 1: most significant half
        spec[t] = make_spec(pos + hi_n, lo_n);          // pass 0
    }
}

// ---------------------------------------------------------------------------
// L1: histogram, per-bin tile scan, bin starts, stable scatter
// ---------------------------------------------------------------------------
// mode 0: digit = spec's digit.  mode 1 (wide keys, speculative): digit = the top
// b1 bits of the W-bit key, and the key OR / complement-OR per table are
// accumulated for the varying-bit mask in the same read.  mode 2: redo mode 1's
// histogram with the spec digit, only for tables whose varying top bits are not the
// top b1 bits (other CTAs exit at once).
// Grid-stride over the (table, tile) items (item = t * T + tile) so that a gated launch
// (the fixed-capacity path's fallback) is a few hundred CTAs that exit at once.
__global__ void __launch_bounds__(kG1Threads) g1_hist(const uint64_t* __restrict__ keys, int64_t n,
                                                    const L1Spec* __restrict__ spec, int nb1,
                                                    uint32_t* __restrict__ hist, int T, int mode, int W, int b1,
                                                    unsigned long long* __restrict__ vm,
                                                    const uint32_t* __restrict__ gate = nullptr, int L = 0) {
    extern __shared__ uint32_t g1_cnt[];
    if (gate && *gate == 0u) return;
    for (int64_t item = blockIdx.x; item < (int64_t)T * L; item += gridDim.x) {
        const int t = (int)(item / T), tile = (int)(item % T);
        L1Spec sp;
        if (mode == 1) {
            sp.nbits = b1;
            sp.shift = W - b1;
            sp.below = 0;
        } else {
            sp = spec[t];
            if (mode == 2 && sp.nbits == b1 && sp.shift == W - b1) continue;
        }
        uint64_t o = 0, no = 0;
        __syncthreads();   // the previous item's counters are written out
        for (int i = threadIdx.x; i < nb1; i += kG1Threads) g1_cnt[i] = 0;
        const int64_t t0 = (int64_t)tile * kG1Tile;
        const uint64_t* kt = keys + (int64_t)t * n + t0;
        const int cn = (int)min((int64_t)kG1Tile, n - t0);
        constexpr int R = 16;   // keys per thread per batch
#pragma unroll 1
        for (int b0 = 0; b0 < kG1Tile; b0 += R * kG1Threads) {
            uint64_t k[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int i = b0 + r * kG1Threads + threadIdx.x;
                k[r] = i < cn ? __ldcs(kt + i) : 0ull;
            }
            if (b0 == 0) __syncthreads();   // counters cleared
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int i = b0 + r * kG1Threads + threadIdx.x;
                if (i < cn) {
                    atomicAdd(&g1_cnt[l1_digit(k[r], sp)], 1u);
                    if (mode == 1) {
                        o |= k[r];
                        no |= ~k[r];
                    }
                }
            }
        }
        if (mode == 1) {
#pragma unroll
            for (int sft = 16; sft > 0; sft >>= 1) {
                o |= __shfl_xor_sync(0xffffffffu, o, sft);
                no |= __shfl_xor_sync(0xffffffffu, no, sft);
            }
            if ((threadIdx.x & 31) == 0) {
                atomicOr(vm + 2 * t, (unsigned long long)o);
                atomicOr(vm + 2 * t + 1, (unsigned long long)no);
            }
        }
        __syncthreads();
        uint32_t* row = hist + ((int64_t)t * T + tile) * nb1;
        for (int b = threadIdx.x; b < nb1; b += kG1Threads) row[b] = g1_cnt[b];
    }
}

// One warp per (table, 32 consecutive bins), lane = bin: exclusive running sum over
// the tiles in place (coalesced rows of the tile-major counts), bin totals out.
__global__ void g1_scan(uint32_t* __restrict__ hist, int T, int L, int nb1, uint32_t* __restrict__ tot,
                        const uint32_t* __restrict__ gate = nullptr) {
    if (gate && *gate == 0u) return;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int groups = (nb1 + 31) / 32;
    if (wg >= (int64_t)L * groups) return;
    const int t = (int)(wg / groups), b = (int)(wg % groups) * 32 + lane;
    if (b >= nb1) return;
    uint32_t* col = hist + (int64_t)t * T * nb1 + b;
    uint32_t run = 0;
    int tile = 0;
    for (; tile + 4 <= T; tile += 4) {
        const uint32_t v0 = col[(int64_t)tile * nb1], v1 = col[(int64_t)(tile + 1) * nb1],
                       v2 = col[(int64_t)(tile + 2) * nb1], v3 = col[(int64_t)(tile + 3) * nb1];
        col[(int64_t)tile * nb1] = run;
        col[(int64_t)(tile + 1) * nb1] = run + v0;
        col[(int64_t)(tile + 2) * nb1] = run + v0 + v1;
        col[(int64_t)(tile + 3) * nb1] = run + v0 + v1 + v2;
        run += v0 + v1 + v2 + v3;
    }
    for (; tile < T; ++tile) {
        const uint32_t v = col[(int64_t)tile * nb1];
        col[(int64_t)tile * nb1] = run;
        run += v;
    }
    tot[(int64_t)t * nb1 + b] = run;
}

// One block per table: bin starts = exclusive scan of the bin totals; with a big-bin
// list (wide keys), every bin larger than kG2BinCap is appended as t * nb1 + bin.
__global__ void __launch_bounds__(1024) g1_binstart(const uint32_t* __restrict__ tot, int nb1, int64_t n,
                                                    uint32_t* __restrict__ binstart, uint32_t* __restrict__ biglist,
                                                    uint32_t* __restrict__ bigcount,
                                                    const uint32_t* __restrict__ gate = nullptr) {
    __shared__ uint32_t ws[32];
    if (gate && *gate == 0u) return;
    const int t = blockIdx.x;
    const int b0 = 2 * threadIdx.x, b1 = b0 + 1;
    const uint32_t v0 = b0 < nb1 ? tot[(int64_t)t * nb1 + b0] : 0u;
    const uint32_t v1 = b1 < nb1 ? tot[(int64_t)t * nb1 + b1] : 0u;
    const uint32_t e = block_excl_scan<1024>(v0 + v1, ws, nullptr);
    uint32_t* bs = binstart + (int64_t)t * (nb1 + 1);
    if (b0 < nb1) bs[b0] = e;
    if (b1 < nb1) bs[b1] = e + v0;
    if (threadIdx.x == 0) bs[nb1] = (uint32_t)n;
    if (!biglist) return;
    if (b0 < nb1 && v0 > (uint32_t)kG2BinCap) biglist[atomicAdd(bigcount, 1u)] = (uint32_t)t * nb1 + b0;
    if (b1 < nb1 && v1 > (uint32_t)kG2BinCap) biglist[atomicAdd(bigcount, 1u)] = (uint32_t)t * nb1 + b1;
}

// Fixed-capacity path (wide keys): bin starts from the bins' final cursors (= their
// sizes) and the digit spec (the top b1 key bits), unless a bin overflowed.
__global__ void __launch_bounds__(1024) g1_fixscan(const uint32_t* __restrict__ cur, int nb1, int64_t n,
                                                   uint32_t* __restrict__ binstart, L1Spec* __restrict__ spec,
                                                   int b1, int W, const uint32_t* __restrict__ ovf,
                                                   uint32_t* __restrict__ hint) {
    __shared__ uint32_t ws[32];
    const uint32_t o = *ovf;
    if (hint && blockIdx.x == 0 && threadIdx.x == 0) {
        const uint32_t h = *hint;
        *hint = (o & 1u) ? 8u : (h > 0u ? h - 1u : 0u);   // real overflow: 8 builds on the histogram path
    }
    if (o) return;
    const int t = blockIdx.x;
    const int b0 = 2 * threadIdx.x, b1i = b0 + 1;
    const uint32_t v0 = b0 < nb1 ? cur[(int64_t)t * nb1 + b0] : 0u;
    const uint32_t v1 = b1i < nb1 ? cur[(int64_t)t * nb1 + b1i] : 0u;
    const uint32_t e = block_excl_scan<1024>(v0 + v1, ws, nullptr);
    uint32_t* bs = binstart + (int64_t)t * (nb1 + 1);
    if (b0 < nb1) bs[b0] = e;
    if (b1i < nb1) bs[b1i] = e + v0;
    if (threadIdx.x == 0) {
        bs[nb1] = (uint32_t)n;
        int pos[12];
        for (int j = 0; j < b1; ++j) pos[j] = W - 1 - j;
        spec[t] = make_spec(pos, b1);
    }
}

// Stable scatter by the L1 digit, persistent: CTA c takes work items c, c + grid, ...
// (item = (table, 4096-key tile), table-major so that the CTAs in flight scatter into
// one table's destination, which stays resident in L2).  A tile's keys are 32 KB
// contiguous: one bulk async copy (cp.async.bulk + mbarrier) per tile into a ring of
// NST shared-memory stages, issued NST-1 tiles ahead, so no thread waits on DRAM.
// Ranking: warp w owns items [256w, 256w+256) in 8 coalesced rounds; match_any gives
// the rank among equal digits in a round, warp-private running counts order the
// rounds, one block pass turns (digit, warp) counts into offsets.  The write-out goes
// through a u16 permutation so consecutive threads write consecutive addresses.
namespace {
__device__ __forceinline__ uint32_t g_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void g_mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(g_smem_u32(bar)));
}
__device__ __forceinline__ void g_mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(g_smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void g_mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LAB_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra LAB_WAIT_%=;\n"
        "}\n" ::"r"(g_smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void g_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(g_smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(g_smem_u32(bar))
        : "memory");
}
}  // namespace

#ifndef LSHB_SCATTER_T
#define LSHB_SCATTER_T 512   // L1 scatter CTA threads
#endif
#ifndef LSHB_SCATTER_NST
#define LSHB_SCATTER_NST 2   // L1 scatter tile ring stages
#endif
constexpr int kSThreads = LSHB_SCATTER_T;
constexpr int kSMaxDPT = (2048 + kSThreads - 1) / kSThreads;   // digits per thread (nb1 <= 2048)
constexpr int kSWarps = kSThreads / 32;
constexpr int kSRounds = kG1Tile / kSThreads;   // 16 at 512 threads

size_t g1_scatter_smem(int nb1, bool stable, int nst) {
    // ring, staged permutation + digit, offsets, counters (per warp if stable)
    return 64 + (size_t)nst * kG1Tile * 8 + (size_t)kG1Tile * 4 + (size_t)nb1 * 8 +
           (stable ? (size_t)kSWarps * nb1 * 2 : (size_t)nb1 * 4);
}

// STABLE = false (wide-key MSD pass): ranks inside a digit come from one shared
// atomicAdd per key (order inside a tile's run of a digit is then arbitrary; the
// per-chunk sort orders ties by id).  STABLE = true (narrow-key LSD passes, which
// need stability): warp-private counts + ballot digit match.
// FIX (wide keys, no histogram pass): the digit is the top b1 key bits and every L1 bin
// has a fixed capacity kG2BinCap in the output ([L][nb1][cap] layout, table stride
// ostride); a tile reserves its run of each digit with one atomicAdd on the bin's
// cursor (cursor[t][d] in `hist`).  A bin that would exceed its capacity sets
// *ovf and its runs are dropped: the histogram path then redoes the grouping.
// (Fingerprint keys are uniform: a C4 bin holds 977 +- 31 keys, cap 1280.)
template <bool IMPLICIT_IDS, bool STABLE, bool FIX = false>
__global__ void __launch_bounds__(kSThreads, LSHB_SCATTER_CPS)
    g1_scatter(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ iin, uint64_t* __restrict__ kout,
               uint32_t* __restrict__ iout, int64_t n, const L1Spec* __restrict__ spec, int nb1,
               const uint32_t* __restrict__ hist, const uint32_t* __restrict__ binstart, int T, int L,
               uint32_t id_base, int nst, const uint32_t* __restrict__ gate = nullptr, uint32_t* __restrict__ ovf = nullptr,
               int fix_b1 = 0, int fix_w = 64, int64_t ostride = 0, const uint32_t* __restrict__ gate_skip = nullptr) {
    extern __shared__ __align__(128) unsigned char g1_dsm[];
    if (gate && *gate == 0u) return;
    if (FIX && gate_skip && *gate_skip) {   // hinted: leave it to the histogram path
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(ovf, 2u);
        return;
    }
    uint64_t* bars = reinterpret_cast<uint64_t*>(g1_dsm);                                  // [nst]
    uint64_t* rk = reinterpret_cast<uint64_t*>(g1_dsm + 64);                               // [nst][4096]
    uint32_t* sp = reinterpret_cast<uint32_t*>(rk + (size_t)nst * kG1Tile);                // staged item | digit << 16
    uint32_t* gpos = sp + kG1Tile;                                                         // [nb1] global - local start
    uint32_t* loc = gpos + nb1;                                                            // [nb1]
    uint16_t* wrun = reinterpret_cast<uint16_t*>(loc + nb1);                               // [kSWarps][nb1]
    __shared__ uint32_t ws[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) g_mbar_init(bars + i);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // bulk copies need 16-byte aligned, 16-byte multiple ranges: full tiles of tables
    // whose base is 16-byte aligned; other tiles are loaded by all threads after the wait
    auto bulk_ok = [&](int t, int tile) {
        const int64_t cnt = min((int64_t)kG1Tile, n - (int64_t)tile * kG1Tile);
        const uint64_t a = reinterpret_cast<uint64_t>(kin + (int64_t)t * n + (int64_t)tile * kG1Tile);
        return cnt == kG1Tile && (a & 15) == 0;
    };
    // work-item cursors advanced incrementally (no 64-bit division per item):
    // item w = blockIdx.x + it * grid  ->  (table t, tile), t-major
    struct Cur {
        int t, tile;
    };
    auto advance = [&](Cur& c) {
        c.tile += gridDim.x;
        while (c.tile >= T) {
            c.tile -= T;
            ++c.t;
        }
    };
    Cur ci{(int)(blockIdx.x / T), (int)(blockIdx.x % T)};   // next item to issue (thread 0)
    int ist = 0;
    auto issue = [&]() {  // thread 0: bulk copy of item ci into stage ist, then advance
        if (ci.t < L) {
            if (!bulk_ok(ci.t, ci.tile)) {
                g_mbar_arrive_tx(bars + ist, 0u);
            } else {
                const int64_t off = (int64_t)ci.t * n + (int64_t)ci.tile * kG1Tile;
                g_mbar_arrive_tx(bars + ist, kG1Tile * 8u);
                g_bulk(rk + (size_t)ist * kG1Tile, kin + off, kG1Tile * 8u, bars + ist);
            }
        }
        advance(ci);
        if (++ist == nst) ist = 0;
    };
    if (threadIdx.x == 0)
        for (int i = 0; i < nst - 1; ++i) issue();

    Cur cc{(int)(blockIdx.x / T), (int)(blockIdx.x % T)};   // item being processed
    int st = 0;
    uint32_t phase = 0;
    for (;; advance(cc)) {
        if (cc.t >= L) break;
        const int t = cc.t, tile = cc.tile;
        L1Spec sp0;
        if constexpr (FIX) {
            sp0.nbits = fix_b1;
            sp0.shift = fix_w - fix_b1;
            sp0.below = 0;
        } else {
            sp0 = spec[t];
        }
        const int64_t tb = (int64_t)t * (FIX ? ostride : n);   // output table base
        const int64_t ti = (int64_t)t * n;                      // input table base
        const int cnt = (int)min((int64_t)kG1Tile, n - (int64_t)tile * kG1Tile);
        uint64_t* kr = rk + (size_t)st * kG1Tile;
        const uint32_t* ir = IMPLICIT_IDS ? nullptr : iin + ti + (int64_t)tile * kG1Tile;
        // this tile's global run starts per digit.  Stable (LSD) passes: loads issued now,
        // consumed after the ranking (measured: SRP scatter 1.39 -> 1.34 ms); the wide-key
        // pass loads them after the scan (prefetching there measured slower, 0.45 -> 0.55 ms)
        const int DPT = (nb1 + kSThreads - 1) / kSThreads;   // <= kSMaxDPT (nb1 <= 2048)
        uint32_t gp[kSMaxDPT];
#pragma unroll
        for (int j = 0; j < kSMaxDPT; ++j) {
            const int d = threadIdx.x * DPT + j;
            gp[j] = (STABLE && j < DPT && d < nb1)
                        ? __ldg(binstart + (int64_t)t * (nb1 + 1) + d) + __ldg(hist + ((int64_t)t * T + tile) * nb1 + d)
                        : 0u;
        }
        g_mbar_wait(bars + st, phase);
        for (int i = threadIdx.x; i < (STABLE ? kSWarps * nb1 : 2 * nb1); i += kSThreads) wrun[i] = 0;
        if (!bulk_ok(t, tile)) {
            for (int i = threadIdx.x; i < cnt; i += kSThreads) kr[i] = kin[ti + (int64_t)tile * kG1Tile + i];
        }
        __syncthreads();   // tile in smem; previous write-out finished with its stage
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue();   // into the stage the previous item used
        }
        if (++st == nst) {
            st = 0;
            phase ^= 1u;
        }
        uint32_t slot[kSRounds];
        const int base = warp * (kG1Tile / kSWarps);
        if constexpr (STABLE) {
            uint16_t* my = wrun + warp * nb1;
            uint32_t peers[kSRounds];
#pragma unroll
            for (int r = 0; r < kSRounds; ++r) {
                const int i = base + r * 32 + lane;
                slot[r] = i < cnt ? l1_digit(kr[i], sp0) : 0x10000u + lane;
                // match.any: cheap when a warp sees few distinct digits (narrow,
                // duplicate-heavy keys take this stable path)
                peers[r] = __match_any_sync(0xffffffffu, slot[r]);
            }
#pragma unroll
            for (int r = 0; r < kSRounds; ++r) {
                const uint32_t dg = slot[r];
                const bool valid = dg < 0x10000u;
                const uint32_t rank = __popc(peers[r] & lanemask_lt());
                const uint32_t before = valid ? my[dg] : 0u;
                __syncwarp();
                if (valid && rank == 0) my[dg] = (uint16_t)(before + __popc(peers[r]));
                __syncwarp();
                slot[r] = (dg << 16) | (before + rank);
            }
        } else {
            uint32_t* c32 = reinterpret_cast<uint32_t*>(wrun);   // [nb1] tile counts
#pragma unroll
            for (int r = 0; r < kSRounds; ++r) {
                const int i = base + r * 32 + lane;
                if (i < cnt) {
                    const uint32_t dg = l1_digit(kr[i], sp0);
                    slot[r] = (dg << 16) | atomicAdd(&c32[dg], 1u);
                }
            }
        }
        __syncthreads();
        // per digit: exclusive over warps (in place), tile count; exclusive over digits -> loc
        // FIX: the bin-cursor atomics are issued as soon as the tile's digit counts are
        // known and their results consumed only after the scan and the placement below,
        // so their latency overlaps both
        uint32_t mysum = 0;
        uint32_t gj[kSMaxDPT], cj[kSMaxDPT];
#pragma unroll
        for (int j = 0; j < kSMaxDPT; ++j) gj[j] = cj[j] = 0u;
        if constexpr (FIX) {
#pragma unroll
            for (int j = 0; j < kSMaxDPT; ++j) {
                const int d = threadIdx.x * DPT + j;
                if (j < DPT && d < nb1) {
                    const uint32_t acc = reinterpret_cast<const uint32_t*>(wrun)[d];
                    if (acc) gj[j] = atomicAdd(const_cast<uint32_t*>(hist) + (int64_t)t * nb1 + d, acc);
                    cj[j] = acc;
                    mysum += acc;
                }
            }
        } else {
            for (int j = 0; j < DPT; ++j) {
                const int d = threadIdx.x * DPT + j;
                if (d < nb1) {
                    uint32_t acc = 0;
                    if constexpr (STABLE) {
#pragma unroll
                        for (int ww = 0; ww < kSWarps; ++ww) {
                            const uint32_t c = wrun[ww * nb1 + d];
                            wrun[ww * nb1 + d] = (uint16_t)acc;
                            acc += c;
                        }
                    } else {
                        acc = reinterpret_cast<const uint32_t*>(wrun)[d];
                    }
                    loc[d] = acc;
                    mysum += acc;
                }
            }
        }
        uint32_t ex = block_excl_scan<kSThreads>(mysum, ws, nullptr);
        // digit starts (loc) and the tile's global run starts: gpos[d] = global start -
        // local start (pos = gpos + p); an overflowed bin gets 0x80000000 (pos out of
        // range: skipped, redone by the fallback)
        uint32_t lj[kSMaxDPT];
#pragma unroll
        for (int j = 0; j < kSMaxDPT; ++j) {
            const int d = threadIdx.x * DPT + j;
            lj[j] = ex;
            if (j < DPT && d < nb1) {
                const uint32_t c = FIX ? cj[j] : loc[d];
                loc[d] = ex;
                ex += c;
                if constexpr (FIX) {
                    lj[j] |= c ? 0u : 0x80000000u;   // no items: nothing to place
                } else {
                    gj[j] = STABLE ? gp[j] : binstart[(int64_t)t * (nb1 + 1) + d] + hist[((int64_t)t * T + tile) * nb1 + d];
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kSRounds; ++r) {
            const int i = base + r * 32 + lane;
            if (i < cnt) {
                const uint32_t dg = slot[r] >> 16;
                const uint32_t p = loc[dg] + (STABLE ? (uint32_t)wrun[warp * nb1 + dg] : 0u) + (slot[r] & 0xffffu);
                sp[p] = (uint32_t)i | (dg << 16);
            }
        }
#pragma unroll
        for (int j = 0; j < kSMaxDPT; ++j) {
            const int d = threadIdx.x * DPT + j;
            if (j < DPT && d < nb1) {
                if (FIX && cj[j] && gj[j] + cj[j] > (uint32_t)kG2BinCap) {   // bin overflow
                    atomicOr(ovf, 1u);
                    lj[j] |= 0x80000000u;
                }
                if (FIX && (lj[j] & 0x80000000u)) gpos[d] = 0x80000000u;
                else gpos[d] = (FIX ? (uint32_t)d * kG2BinCap + gj[j] : gj[j]) - lj[j];
            }
        }
        __syncthreads();
        const uint32_t olim = (uint32_t)(FIX ? ostride : n);
        for (int p = threadIdx.x; p < cnt; p += kSThreads) {
            const uint32_t v = sp[p], i = v & 0xffffu, dg = v >> 16;
            const uint32_t pos = gpos[dg] + (uint32_t)p;
            if (FIX && pos >= olim) continue;   // overflowed bin: the fallback redoes it
            if (LSHB_OK(pos < olim && i < (uint32_t)cnt)) {
                kout[tb + pos] = kr[i];
                iout[tb + pos] = IMPLICIT_IDS ? id_base + (uint32_t)(tile * kG1Tile) + i : __ldg(ir + i);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// L2: per-bin sort, run-length encoding and chained bucket numbering (wide keys)
// ---------------------------------------------------------------------------
struct G2Args {
    const uint64_t* keys;       // L1 output [L][n]
    const uint32_t* ids;        // L1 output [L][n]
    const uint32_t* binstart;   // [L][nb1+1]
    unsigned long long* state;  // (unused by the wide-key path)
    uint32_t* scratch;          // [L][2n] permutation ping-pong of bins larger than kG2BinCap
    const L1Spec* spec;         // [L]
    int64_t n;
    int L;
    int nb1;                    // L1 bins per table (= numbering units per table)
    uint32_t id_base;           // ids of a table are id_base + row
    const uint32_t* biglist;    // t * nb1 + bin of every bin larger than kG2BinCap
    const uint32_t* bigcount;   // [1] entries of biglist
    uint32_t* binheads;         // [L][nb1] buckets per bin (big bins: written by g2_big)
    uint32_t* ticket;           // [1] g2a's dynamic bin counter (zero before the launch)
    const uint32_t* ovf;        // fixed-capacity L1 layout unless *ovf (nullptr: compact layout)
    int64_t fix_tstride;        // fixed layout: table stride of keys / ids (nb1 * kG2BinCap)
    IndexDev out;
};

template <typename PT>
__device__ __forceinline__ uint32_t pget(const PT* p, int64_t r) {
    return p ? (uint32_t)p[r] : (uint32_t)r;
}

// Look-back state words: (flag << 32) | value in ONE aligned 64-bit word, so a reader
// sees flag and value together (single-copy atomicity) and no other data is passed
// through them: relaxed gpu-scope accesses suffice (st.release / ld.acquire compiled to
// MEMBAR.ALL.GPU and an L1 invalidation, CCTL.IVALL, on the bin's critical path).
__device__ __forceinline__ void st_state(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_state(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Decoupled look-back over the bins of one table, one warp: publishes this bin's
// bucket count and returns the number of buckets in all earlier bins.  The warp
// inspects 32 predecessors per step (lane 0 = nearest) and stops at the nearest
// inclusive prefix.  Bins of a table are launched in increasing block order, so
// predecessors are running.
// `pre` (optional): the first round's values, loaded earlier by lookback_preload.
__device__ __forceinline__ unsigned long long lookback_preload(const unsigned long long* st, int b) {
    const int idx = b - 1 - (int)(threadIdx.x & 31);
    return idx >= 0 ? ld_state(st + idx) : (2ull << 32);
}
__device__ uint32_t chained_prefix_warp(unsigned long long* st, int b, uint32_t agg, bool published = false,
                                        const unsigned long long* pre = nullptr) {
    const int lane = threadIdx.x & 31;
    if (lane == 0 && !published) st_state(st + b, ((b == 0 ? 2ull : 1ull) << 32) | agg);
    if (b == 0) return 0;
    uint32_t acc = 0;
    int j = b - 1;
    bool first = pre != nullptr;
    while (true) {
        const int idx = j - lane;
        const unsigned long long v = first ? *pre : idx >= 0 ? ld_state(st + idx) : (2ull << 32);
        first = false;
        const uint32_t f = (uint32_t)(v >> 32);
        const uint32_t incl = __ballot_sync(0xffffffffu, f == 2);
        const uint32_t notready = __ballot_sync(0xffffffffu, f == 0);
        const int first = incl ? __ffs(incl) - 1 : 31;
        const uint32_t need = (first == 31) ? 0xffffffffu : ((2u << first) - 1u);
        if (notready & need) {
            __nanosleep(64);
            continue;
        }
        uint32_t val = (lane <= first) ? (uint32_t)v : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        acc += val;
        if (incl) break;
        j -= 32;
    }
    if (lane == 0) st_state(st + b, (2ull << 32) | (acc + agg));
    return acc;
}

// Bits that vary over K[0..len) (OR ^ AND).
template <typename KE>
__device__ uint64_t cta_varying(const KE* K, int64_t len, unsigned long long* red) {
    if (threadIdx.x == 0) {
        red[0] = 0ull;
        red[1] = ~0ull;
    }
    __syncthreads();
    uint64_t o = 0, a = ~0ull;
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
        const uint64_t k = K[i];
        o |= k;
        a &= k;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, s);
        a &= __shfl_xor_sync(0xffffffffu, a, s);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicOr(&red[0], (unsigned long long)o);
        atomicAnd(&red[1], (unsigned long long)a);
    }
    __syncthreads();
    const uint64_t v = len > 0 ? (red[0] ^ red[1]) : 0ull;
    __syncthreads();
    return v;
}

// Stable counting pass on the 8-bit digit at `sh` of K[src[i]], i < len; dst
// receives src in digit order (src == nullptr: identity).  Warps own contiguous
// ranges; per-warp digit counts -> (digit, warp) offsets -> ranked scatter.
struct ShiftDigit {
    int sh;
    __device__ __forceinline__ uint32_t operator()(uint64_t k) const { return (uint32_t)(k >> sh) & 255u; }
};
template <typename PT, typename CT, typename DF = ShiftDigit, typename KE = uint64_t>
__device__ void cta_digit_pass(const KE* K, const PT* src, PT* dst, int64_t len, DF df, CT* wcnt,
                               uint32_t* ws) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t per = ((len + kG2Warps - 1) / kG2Warps + 31) / 32 * 32;
    const int64_t a0 = min(len, (int64_t)warp * per), a1 = min(len, a0 + per);
    for (int i = threadIdx.x; i < kG2Warps * 256; i += kG2Threads) wcnt[i] = 0;
    __syncthreads();
    CT* my = wcnt + warp * 256;
    for (int64_t b = a0; b < a1; b += 32) {
        const int64_t i = b + lane;
        const bool valid = i < a1;
        const uint32_t s = valid ? pget(src, i) : 0u;
        const uint32_t dg = valid ? df(K[s]) : 256u + lane;
        const uint32_t peers = match_digit<8>(dg, 8, valid);
        if (valid && (peers & lanemask_lt()) == 0) my[dg] = (CT)(my[dg] + __popc(peers));
        __syncwarp();
    }
    __syncthreads();
    {
        const int d = threadIdx.x;
        uint32_t tot = 0;
        if (d < 256)
            for (int w = 0; w < kG2Warps; ++w) tot += wcnt[w * 256 + d];
        uint32_t acc = block_excl_scan<kG2Threads>(tot, ws, nullptr);
        if (d < 256)
            for (int w = 0; w < kG2Warps; ++w) {
                const uint32_t c = wcnt[w * 256 + d];
                wcnt[w * 256 + d] = (CT)acc;
                acc += c;
            }
    }
    __syncthreads();
    for (int64_t b = a0; b < a1; b += 32) {
        const int64_t i = b + lane;
        const bool valid = i < a1;
        const uint32_t s = valid ? pget(src, i) : 0u;
        const uint32_t dg = valid ? df(K[s]) : 256u + lane;
        const uint32_t peers = match_digit<8>(dg, 8, valid);
        const uint32_t rank = __popc(peers & lanemask_lt());
        const uint32_t before = valid ? (uint32_t)my[dg] : 0u;
        __syncwarp();
        if (valid) {
            dst[before + rank] = (PT)s;
            if (rank == 0) my[dg] = (CT)(before + __popc(peers));
        }
        __syncwarp();
    }
    __syncthreads();
}

// LSD passes over the 8-bit digits below `top` that vary (bit set in `varying`);
// the permutation starts in *cur (nullptr = identity) and ends in *cur.  Both
// ping-pong buffers are [len].
template <typename PT, typename CT, typename KE = uint64_t>
__device__ void cta_lsd(const KE* K, PT*& cur, PT* b0, PT* b1, int64_t len, int top, uint64_t varying, CT* wcnt,
                        uint32_t* ws) {
    for (int sh = 0; sh < top; sh += 8) {
        const uint64_t dmask = (top - sh >= 8 ? 0xffull : ((1ull << (top - sh)) - 1)) << sh;
        if ((varying & dmask) == 0) continue;
        PT* dst = (cur == b0) ? b1 : b0;
        cta_digit_pass<PT, CT, ShiftDigit, KE>(K, cur, dst, len, ShiftDigit{sh}, wcnt, ws);
        cur = dst;
    }
}

// Order a permutation range by id when its items are in L1 order: the wide-key L1
// pass writes each tile's items of a bin as one run, bins in order and tiles in
// order inside a bin, ids shuffled inside a run.  Along any stable sub-range the run
// id (L1 bin, tile) is non-decreasing; every maximal run is sorted by the low 13 id
// bits with an 8192-bit bitmap.  src -> dst (both [len], global).
__device__ void cta_sort_tile_runs(const uint32_t* ID, const uint64_t* K, const L1Spec& sp, const uint32_t* src,
                                   uint32_t* dst, int64_t len, uint32_t id_base, uint32_t* bm /*[256]*/,
                                   uint16_t* loc /*[8192]*/, uint32_t* ws) {
    auto run_of = [&](int64_t r) {
        const uint32_t p = pget(src, r);
        return ((uint64_t)l1_digit(K[p], sp) << 32) | ((ID[p] - id_base) >> 13);
    };
    int64_t start = 0;
    while (start < len) {
        const uint64_t run = run_of(start);
        int64_t a0 = start + 1, b0 = len;
        while (a0 < b0) {
            const int64_t mid = (a0 + b0) >> 1;
            if (run_of(mid) == run) a0 = mid + 1;
            else b0 = mid;
        }
        const int64_t end = a0;
        for (int w = threadIdx.x; w < 256; w += kG2Threads) bm[w] = 0u;
        __syncthreads();
        for (int64_t r = start + threadIdx.x; r < end; r += kG2Threads) {
            const uint32_t b = (ID[pget(src, r)] - id_base) & 8191u;
            atomicOr(&bm[b >> 5], 1u << (b & 31u));
            loc[b] = (uint16_t)(r - start);
        }
        __syncthreads();
        const uint32_t c = threadIdx.x < 256 ? (uint32_t)__popc(bm[threadIdx.x]) : 0u;
        const uint32_t ex = block_excl_scan<kG2Threads>(c, ws, nullptr);
        if (threadIdx.x < 256) {
            uint32_t bits = bm[threadIdx.x];
            int64_t o = start + ex;
            while (bits) {
                const int b = __ffs(bits) - 1;
                dst[o++] = pget(src, start + loc[threadIdx.x * 32 + b]);
                bits &= bits - 1u;
            }
        }
        __syncthreads();
        start = end;
    }
    __threadfence_block();
    __syncthreads();
}

// Bins larger than kG2BinCap (skewed codes: many equal keys), on global memory: a
// stable 3-way split around a dominant key, id order by tile runs, then stable 8-bit
// passes over the varying key digits.  The sorted permutation ends in p0 (scratch).
__device__ void big_bin_sort(const G2Args& a, int t, int64_t lo, int64_t len, unsigned char* g2_dsm, uint32_t* ws,
                             unsigned long long* red, uint32_t* cls_cnt) {
    const int64_t n = a.n;
    const uint64_t* gk = a.keys + (int64_t)t * n + lo;
    const uint32_t* gi = a.ids + (int64_t)t * n + lo;
    const L1Spec sp = a.spec[t];
    uint32_t* wc = reinterpret_cast<uint32_t*>(g2_dsm);  // [kG2Warps][256] u32
    uint32_t* p0 = a.scratch + (int64_t)t * 2 * n + lo;
    uint32_t* p1 = p0 + n;
    // (key, id) order: the L1 pass does not keep ids ordered inside a bin
    const uint64_t varying = cta_varying(gk, len, red);
    const int sh1 = varying ? 64 - __clzll((long long)varying) : 0;
    uint32_t* cur = nullptr;
    uint32_t* rbm = reinterpret_cast<uint32_t*>(g2_dsm + 16384);          // [256]
    uint16_t* rloc = reinterpret_cast<uint16_t*>(g2_dsm + 16384 + 1024);   // [8192]
    if (!varying) {
        // one bucket: order by id (tile runs, bitmap per run)
        cta_sort_tile_runs(gi, gk, sp, nullptr, p0, len, a.id_base, rbm, rloc, ws);
        cur = p0;
    } else {
        // stable 3-way split around the key at the middle position when it dominates
        const uint64_t pivot = gk[len / 2];
        if (threadIdx.x < 3) cls_cnt[threadIdx.x] = 0;
        __syncthreads();
        uint32_t lt = 0, eq = 0;
        for (int64_t i = threadIdx.x; i < len; i += kG2Threads) {
            const uint64_t k = gk[i];
            lt += k < pivot;
            eq += k == pivot;
        }
        atomicAdd(&cls_cnt[0], lt);
        atomicAdd(&cls_cnt[1], eq);
        __syncthreads();
        const int64_t nlt = cls_cnt[0], neq = cls_cnt[1];
        __syncthreads();
        if (neq * 4 >= len) {
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
            uint32_t base0 = 0, base1 = (uint32_t)nlt, base2 = (uint32_t)(nlt + neq);
            for (int64_t b0 = 0; b0 < len; b0 += kG2Threads) {
                const int64_t i = b0 + threadIdx.x;
                const bool valid = i < len;
                const uint64_t k = valid ? gk[i] : 0ull;
                const uint32_t cls = !valid ? 3u : (k < pivot ? 0u : (k == pivot ? 1u : 2u));
                const uint32_t m0 = __ballot_sync(0xffffffffu, cls == 0), m1 = __ballot_sync(0xffffffffu, cls == 1),
                               m2 = __ballot_sync(0xffffffffu, cls == 2);
                if (lane == 0) {
                    wc[warp * 3] = __popc(m0);
                    wc[warp * 3 + 1] = __popc(m1);
                    wc[warp * 3 + 2] = __popc(m2);
                }
                __syncthreads();
                uint32_t q0 = base0, q1 = base1, q2 = base2;
                for (int w = 0; w < warp; ++w) {
                    q0 += wc[w * 3];
                    q1 += wc[w * 3 + 1];
                    q2 += wc[w * 3 + 2];
                }
                const uint32_t lm = lanemask_lt();
                if (valid) {
                    const uint32_t pos = cls == 0 ? q0 + __popc(m0 & lm) : cls == 1 ? q1 + __popc(m1 & lm)
                                                                                    : q2 + __popc(m2 & lm);
                    p0[pos] = (uint32_t)i;
                }
                for (int w = 0; w < kG2Warps; ++w) {
                    base0 += wc[w * 3];
                    base1 += wc[w * 3 + 1];
                    base2 += wc[w * 3 + 2];
                }
                __syncthreads();
            }
            __threadfence_block();
            __syncthreads();
            // each part by id; the less / greater parts then by key (stable passes)
            const int64_t part_lo[3] = {0, nlt, nlt + neq};
            const int64_t part_len[3] = {nlt, neq, len - nlt - neq};
            for (int q = 0; q < 3; ++q) {
                if (part_len[q] <= 1) continue;
                uint32_t* c = p0 + part_lo[q];
                // the stable partition kept the tile-run structure: id order by tile runs
                cta_sort_tile_runs(gi, gk, sp, c, p1 + part_lo[q], part_len[q], a.id_base, rbm, rloc, ws);
                c = p1 + part_lo[q];
                if (q != 1)
                    cta_lsd<uint32_t, uint32_t>(gk, c, p0 + part_lo[q], p1 + part_lo[q], part_len[q], sh1, varying, wc,
                                                ws);
                if (c != p0 + part_lo[q]) {
                    for (int64_t r = threadIdx.x; r < part_len[q]; r += kG2Threads) p0[part_lo[q] + r] = c[r];
                    __threadfence_block();
                    __syncthreads();
                }
            }
            cur = p0;
        } else {
            cta_sort_tile_runs(gi, gk, sp, nullptr, p0, len, a.id_base, rbm, rloc, ws);
            cur = p0;
            cta_lsd<uint32_t, uint32_t>(gk, cur, p0, p1, len, sh1, varying, wc, ws);
        }
    }
    if (cur != p0) {
        for (int64_t r = threadIdx.x; r < len; r += kG2Threads) p0[r] = cur[r];
        __threadfence_block();
        __syncthreads();
    }
}

// Big bins: sort (permutation in p0), write the bin's ids in final order and its
// bucket count; g2a emits its ukeys / offs through the permutation.  Persistent over
// the big-bin list.
__global__ void __launch_bounds__(kG2Threads) g2_big(G2Args a) {
    extern __shared__ __align__(16) unsigned char g2_dsm[];
    __shared__ uint32_t ws[32];
    __shared__ unsigned long long red[2];
    __shared__ uint32_t cls_cnt[3];
    const uint32_t cnt = *a.bigcount;
    for (uint32_t i = blockIdx.x; i < cnt; i += gridDim.x) {
        const uint32_t e = a.biglist[i];
        const int t = (int)(e / (uint32_t)a.nb1), bin = (int)(e % (uint32_t)a.nb1);
        const uint32_t* bs = a.binstart + (int64_t)t * (a.nb1 + 1);
        const int64_t lo = bs[bin], len = (int64_t)bs[bin + 1] - lo;
        if (threadIdx.x == 0) {
            red[0] = 0ull;
            red[1] = ~0ull;
        }
        __syncthreads();
        big_bin_sort(a, t, lo, len, g2_dsm, ws, red, cls_cnt);
        const uint64_t* gk = a.keys + (int64_t)t * a.n + lo;
        const uint32_t* gi = a.ids + (int64_t)t * a.n + lo;
        const uint32_t* p0 = a.scratch + (int64_t)t * 2 * a.n + lo;
        uint32_t* od = a.out.ids + (int64_t)t * a.n + lo;
        uint32_t heads = 0;
        for (int64_t r = threadIdx.x; r < len; r += kG2Threads) {
            const uint32_t pr = p0[r];
            if (LSHB_OK(pr < (uint32_t)len)) od[r] = gi[pr];
            heads += (r == 0 || gk[p0[r - 1]] != gk[pr]) ? 1u : 0u;
        }
        uint32_t tot;
        block_excl_scan<kG2Threads>(heads, ws, &tot);
        if (threadIdx.x == 0) a.binheads[(int64_t)t * a.nb1 + bin] = tot;
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// g2a: one CTA (4 warps) per L1 bin of <= kG2aCap items (larger: g2_big), no
// cross-bin dependency, many CTAs resident per SM.  In shared memory:
//   (1) counting scatter on the D <= 12 key bits right below the L1 digit (the keys
//       of a bin agree on every bit above), ranks from the counting atomics;
//   (2) a digit holding one item (for fingerprints ~3/4 of them) places it at its
//       final position at once; the items of a shared digit are ranked among its
//       members by (key, id), and segments longer than kG2aLong (duplicate-heavy
//       codes) are bitonic-sorted; a bucket head is an item with no equal key of
//       smaller id;
//   (3) ids stream out coalesced;
//   (4) the bin's bucket count is published for a decoupled look-back over the bins of
//       its table (dynamic ticket order); warp 0 looks back while the others write
//       the ids, then ukeys / offs are written at their final, compacted positions.
// ---------------------------------------------------------------------------
constexpr int kG2aT = LSHB_G2_T;
constexpr int kG2aW = kG2aT / 32;
constexpr int kG2aIPT = LSHB_G2_IPT;
constexpr int kG2aCap = kG2aT * kG2aIPT;      // 1280 items
constexpr int kG2aD = LSHB_G2_D;               // digit bits (2^D counters)
constexpr int kG2aCW = 1 << (kG2aD - 1);       // counter words (two u16 counters each)
#ifndef LSHB_G2_LONG
#define LSHB_G2_LONG 64
#endif
constexpr int kG2aLong = LSHB_G2_LONG;         // longest segment ranked item by item (O(s^2), worklist)
constexpr int kG2aLongMax = kG2aCap / kG2aLong;
constexpr int kG2aP2 = kG2aCap <= 1024 ? 1024 : kG2aCap <= 2048 ? 2048 : 4096;   // bitonic width >= cap
// digit counters, then (after the placement) the long-segment scratch:
// perm [kG2aP2] u16 | fin [kG2aCap] u16 | off [kG2aLongMax + 1] u32
constexpr int kG2aScratchW = (kG2aP2 * 2 + kG2aCap * 2 + (kG2aLongMax + 1) * 4 + 3) / 4;
constexpr int kG2aCntW = kG2aCW > kG2aScratchW ? kG2aCW : kG2aScratchW;
static_assert(kG2aCap == kG2BinCap, "big-bin threshold");

// Barrier of the per-bin sort: named barrier 1 over its 128 sorting threads (a
// persistent variant with a producer warp that never joins it was measured slower:
// C4 g2 1.25 vs 0.91 ms — fewer CTAs per SM hide less of the sort's own latency).
__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, %0;" ::"n"(kG2aT) : "memory"); }
__device__ __forceinline__ void g_mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(g_smem_u32(bar)) : "memory");
}
// Exclusive scan of one value per consumer thread (128), with total.
__device__ __forceinline__ uint32_t cblock_excl_scan(uint32_t v, uint32_t* ws, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    cbar();
    uint32_t before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < kG2aW; ++w) {
        const uint32_t c = ws[w];
        before += w < warp ? c : 0u;
        all += c;
    }
    if (total) *total = all;
    cbar();
    return before + x - v;
}

struct __align__(16) G2aSmem {
    uint64_t sk[kG2aCap];
    uint32_t si[kG2aCap];
    uint32_t cnt[kG2aCntW];   // digit counters -> digit starts -> final positions (fin) + long-segment scratch
    uint32_t wl[kG2aCap];   // short-segment worklist: p | s0 << 12 | len << 24
    uint32_t ws[kG2aW];
    uint32_t lseg[kG2aLongMax];
    uint32_t nlong, heads, nwl;
};
static_assert(kG2aCap <= 4096 && kG2aLong <= 127, "worklist packing");
static_assert(kG2aLongMax <= kG2aT, "long segments: one per thread when ordering them");

// Bitonic sort of the items at [s0, s0 + len) of S by (key, id): fin[p] = final
// position of the item at p, bit 15 = bucket head.
// All segments longer than kG2aLong (duplicate-heavy codes) in ONE bitonic network:
// their items (the union of the ranges S.lseg[0..nl), s0 << 16 | len) sorted by
// (key, id); since distinct segments hold distinct digits (key ranges), the j-th item
// of the sorted union belongs at the j-th position of the union in increasing order.
// fin[p] = final position of the item at p, bit 15 = bucket head.  S.lseg is sorted
// by s0 in place; `off` [kG2aLongMax + 1] receives the ranges' prefix lengths.
__device__ void g2a_long_union(G2aSmem& S, uint32_t nl, uint16_t* perm, uint16_t* fin, uint32_t* off) {
    // order the ranges by start (nl <= kG2aLongMax): rank by count of smaller starts
    const uint32_t g = threadIdx.x;   // nl <= kG2aLongMax <= kG2aT: one range per thread
    uint32_t r = 0, v = 0;
    if (g < nl) {
        v = S.lseg[g];
        for (uint32_t h = 0; h < nl; ++h) r += S.lseg[h] < v ? 1u : 0u;
    }
    cbar();
    if (g < nl) S.lseg[r] = v;
    cbar();
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (uint32_t g = 0; g < nl; ++g) {
            off[g] = acc;
            acc += S.lseg[g] & 0xffffu;
        }
        off[nl] = acc;
    }
    cbar();
    const int total = (int)off[nl];
    int P = 1;
    while (P < total) P <<= 1;
    // position of the j-th union item (binary search over the range offsets)
    auto upos = [&](int j) {
        uint32_t lo = 0, hi = nl;   // last range with off <= j
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (off[mid] <= (uint32_t)j) lo = mid;
            else hi = mid;
        }
        return (S.lseg[lo] >> 16) + ((uint32_t)j - off[lo]);
    };
    for (int i = threadIdx.x; i < P; i += kG2aT) perm[i] = (uint16_t)(i < total ? upos(i) : 0xffffu);
    cbar();
    auto less = [&](uint16_t x, uint16_t y) {   // pads (0xffff) sort last
        if (x == 0xffffu) return false;
        if (y == 0xffffu) return true;
        const uint64_t kx = S.sk[x], ky = S.sk[y];
        return kx < ky || (kx == ky && S.si[x] < S.si[y]);
    };
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < (P >> 1); i += kG2aT) {
                const int lo = 2 * stride * (i / stride) + (i % stride), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint16_t x = perm[lo], y = perm[hi];
                if (less(y, x) == up) {
                    perm[lo] = y;
                    perm[hi] = x;
                }
            }
            cbar();
        }
    }
    for (int j = threadIdx.x; j < total; j += kG2aT) {
        const uint16_t pj = perm[j];
        const bool head = j == 0 || S.sk[perm[j - 1]] != S.sk[pj];
        fin[pj] = (uint16_t)(upos(j) | (head ? 0x8000u : 0u));
    }
    cbar();
}

// Big bin (sorted by g2_big: ids written, permutation in a.scratch, bucket count in
// binheads): publish, look back, emit its ukeys / offs through the permutation.
__device__ void g2a_big_emit(const G2Args& a, int t, int bin, int64_t lo, int len, uint32_t* s_base) {
    __shared__ uint32_t ws[kG2aW];
    const int nb1 = a.nb1;
    const int64_t n = a.n;
    const uint32_t agg = a.binheads[(int64_t)t * nb1 + bin];
    unsigned long long* st = a.state + (int64_t)t * nb1;
    if (threadIdx.x < 32) {
        const uint32_t pre = chained_prefix_warp(st, bin, agg);
        if (threadIdx.x == 0) *s_base = pre;
    }
    cbar();
    uint32_t b = *s_base;
    const uint64_t* gk = a.keys + (int64_t)t * n + lo;
    const uint32_t* perm = a.scratch + (int64_t)t * 2 * n + lo;
    uint64_t* uk = a.out.ukeys + (int64_t)t * n;
    uint32_t* of = a.out.offs + (int64_t)t * (n + 1);
    for (int p0 = 0; p0 < len; p0 += kG2aT) {
        const int p = p0 + (int)threadIdx.x;
        const uint64_t k = p < len ? gk[perm[p]] : 0ull;
        const bool h = p < len && (p == 0 || k != gk[perm[p - 1]]);
        uint32_t all;
        const uint32_t ex = cblock_excl_scan(h ? 1u : 0u, ws, &all);
        if (h && LSHB_OK((int64_t)b + ex < n)) {
            uk[b + ex] = k;
            of[b + ex] = (uint32_t)(lo + p);
        }
        b += all;
    }
    if (bin == nb1 - 1 && threadIdx.x == 0) {
        a.out.nb[t] = b;
        of[b] = (uint32_t)n;
    }
}

// Sort one L1 bin of len <= kG2aCap items (keys kr, ids ir: item u + j * kG2aT of the
// bin in register j, already loaded by the caller) in shared memory and emit its ids,
// ukeys and offs (module comment above).  Executed by the kG2aT threads of the CTA
// (named barrier 1).
__device__ __forceinline__ void g2_bin(const G2Args& a, G2aSmem& S, int t, int bin, int64_t lo, int len,
                                       const uint64_t (&kr)[kG2aIPT], const uint32_t (&ir)[kG2aIPT],
                                       uint32_t* s_base_p) {
    const int u = threadIdx.x, lane = u & 31, wu = u >> 5;
    const int nb1 = a.nb1;
    const int64_t n = a.n;
    uint32_t dr[kG2aIPT];
    // (the digit counters and S.nlong / S.heads / S.nwl were zeroed by the caller before
    // its last barrier)
    const L1Spec sp = a.spec[t];
    // keys of the bin agree on every bit at or above the lowest L1 digit bit (hb)
    const int hb = sp.below == 0 ? 0 : 64 - __clzll((long long)sp.below);
    const int D = min(kG2aD, hb), sh = hb - D;
    const uint32_t dmask = (1u << D) - 1u;
    // (1) digit counts; the atomic's old value is the item's rank inside its digit
#pragma unroll
    for (int j = 0; j < kG2aIPT; ++j) {
        const int i = u + j * kG2aT;
        if (i < len) {
            const uint32_t d = (uint32_t)(kr[j] >> sh) & dmask;
            const uint32_t hs = (d & 1u) << 4;
            const uint32_t old = atomicAdd(&S.cnt[d >> 1], 1u << hs);
            dr[j] = (d << 16) | ((old >> hs) & 0xffffu);
        }
    }
    cbar();
    {
        // exclusive scan of the 4096 counters: thread u owns words [16u, 16u + 16)
        constexpr int WPT = kG2aCW / kG2aT;
        uint32_t wv[WPT], sum = 0;
        const uint4* c4 = reinterpret_cast<const uint4*>(S.cnt + WPT * u);
#pragma unroll
        for (int q4 = 0; q4 < WPT / 4; ++q4) {
            const uint4 v = c4[q4];
            wv[4 * q4] = v.x;
            wv[4 * q4 + 1] = v.y;
            wv[4 * q4 + 2] = v.z;
            wv[4 * q4 + 3] = v.w;
        }
#pragma unroll
        for (int qq = 0; qq < WPT; ++qq) sum += (wv[qq] & 0xffffu) + (wv[qq] >> 16);
        uint32_t x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) S.ws[wu] = x;
        cbar();
        uint32_t ex = x - sum;
#pragma unroll
        for (int w = 0; w < kG2aW; ++w) ex += w < wu ? S.ws[w] : 0u;
        uint4* o4 = reinterpret_cast<uint4*>(S.cnt + WPT * u);
#pragma unroll
        for (int q4 = 0; q4 < WPT / 4; ++q4) {
            uint32_t o[4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const uint32_t w = wv[4 * q4 + jj], c0 = w & 0xffffu;
                o[jj] = ex | ((ex + c0) << 16);
                ex += c0 + (w >> 16);
            }
            o4[q4] = make_uint4(o[0], o[1], o[2], o[3]);
        }
    }
    cbar();
    // (2) place: an item alone in its digit is final; the others go to their digit's
    // region (arbitrary order) and get their final position from fin[] below.  dr: kDone;
    // a short-segment member's worklist entry p | s0 << 12 | len << 24; a long-segment
    // member's p | kLongBit
    constexpr uint32_t kDone = 0xffffffffu, kLongBit = 0x80000000u;
    uint16_t* fin = reinterpret_cast<uint16_t*>(S.cnt) + kG2aP2;   // [kG2aCap]: final position | head << 15
    uint32_t heads = 0, nshort = 0;
#pragma unroll
    for (int j = 0; j < kG2aIPT; ++j) {
        const int i = u + j * kG2aT;
        if (i < len) {
            const uint32_t d = dr[j] >> 16, r = dr[j] & 0xffffu;
            const uint32_t w0 = S.cnt[d >> 1];
            const uint32_t s0 = (w0 >> ((d & 1u) << 4)) & 0xffffu;
            const uint32_t s1 = d == dmask ? (uint32_t)len
                                           : ((d & 1u) ? (S.cnt[(d + 1) >> 1] & 0xffffu) : (w0 >> 16));
            const uint32_t p = s0 + r;
            if (LSHB_OK(p < (uint32_t)len)) {
                S.sk[p] = kr[j];
                S.si[p] = ir[j];
                if (s1 - s0 == 1) {
                    dr[j] = kDone;
                    ++heads;
                } else if (s1 - s0 <= (uint32_t)kG2aLong) {
                    dr[j] = p | (s0 << 12) | ((s1 - s0) << 24);
                    ++nshort;
                } else {
                    dr[j] = p | kLongBit;
                    if (r == 0) S.lseg[atomicAdd(&S.nlong, 1u)] = (s0 << 16) | (s1 - s0);
                }
            } else {
                dr[j] = kDone;
            }
        }
    }
    {
        // append the short-segment members to the worklist: one warp scan of the
        // per-thread counts and one shared atomic per warp
        uint32_t x = nshort;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        uint32_t wbase = 0;
        if (lane == 31 && x) wbase = atomicAdd(&S.nwl, x);
        wbase = __shfl_sync(0xffffffffu, wbase, 31) + x - nshort;
#pragma unroll
        for (int j = 0; j < kG2aIPT; ++j) {
            const int i = u + j * kG2aT;
            if (i < len && dr[j] != kDone && !(dr[j] & kLongBit)) S.wl[wbase++] = dr[j];
        }
    }
    cbar();
    // rank the worklist (members of digits shared by 2..kG2aLong items) by (key, id)
    // inside their digit: fin[p] = final position, bit 15 = bucket head (no equal key of
    // smaller id).  Reads only sk / si; every thread takes entries, not just the owners.
    {
        const uint32_t nw = S.nwl;
        for (uint32_t w = u; w < nw; w += kG2aT) {
            const uint32_t e = S.wl[w];
            const uint32_t p = e & 0xfffu, s0 = (e >> 12) & 0xfffu, sl = (e >> 24) & 0x7fu;
            const uint64_t k = S.sk[p];
            const uint32_t id = S.si[p];
            uint32_t f = s0, dup = 0;
            for (uint32_t qq = s0; qq < s0 + sl; ++qq) {
                const uint64_t kq = S.sk[qq];
                const uint32_t iq = S.si[qq];
                const bool eq_lt = kq == k && iq < id;
                f += (kq < k || eq_lt) ? 1u : 0u;
                dup |= eq_lt ? 1u : 0u;
            }
            fin[p] = (uint16_t)(f | ((dup ^ 1u) << 15));
        }
    }
    const uint32_t nl = S.nlong;   // complete: appended before the last barrier
    if (nl) {
        // duplicate-heavy segments: bitonic sort by (key, id) in the counter area:
        // perm [kG2aP2] u16 | fin [kG2aCap] u16 | off [kG2aLongMax + 1] u32
        uint16_t* perm = reinterpret_cast<uint16_t*>(S.cnt);
        g2a_long_union(S, nl, perm, fin, reinterpret_cast<uint32_t*>(fin + kG2aCap));
    } else {
        cbar();
    }
    // final positions of the items of shared digits, written at once: every read of sk /
    // si by the ranking is behind the last barrier, and the fin[] reads touch the counter
    // area only
#pragma unroll
    for (int j = 0; j < kG2aIPT; ++j) {
        const int i = u + j * kG2aT;
        if (i < len && dr[j] != kDone) {
            const uint32_t fv = fin[dr[j] & 0xfffu];
            const uint32_t f = fv & 0x7fffu;
            heads += fv >> 15;
            if (LSHB_OK(f < (uint32_t)len)) {
                S.sk[f] = kr[j];
                S.si[f] = ir[j];
            }
        }
    }
    heads = __reduce_add_sync(0xffffffffu, heads);
    if (lane == 0) atomicAdd(&S.heads, heads);
    cbar();   // the bin is sorted in sk / si; S.heads complete
    unsigned long long* st = a.state + (int64_t)t * nb1;
    const uint32_t agg = S.heads;
    if (u == 0) st_state(st + bin, ((bin == 0 ? 2ull : 1ull) << 32) | agg);   // publish
    // (3) ids out (coalesced, by warps 1..) while warp 0 looks back for the bin's first
    // bucket number
    uint32_t* od = a.out.ids + (int64_t)t * n + lo;
    if (u >= 32) {
        for (int p = u - 32; p < len; p += kG2aT - 32) __stcs(od + p, S.si[p]);
    } else {
        const uint32_t pre = chained_prefix_warp(st, bin, agg, /*published=*/true);
        if (u == 0) *s_base_p = pre;
    }
    cbar();
    // (4) ukeys / offs: a head is a key that differs from its predecessor (the first key
    // of a bin always does: bins differ in the L1 digit)
    const uint32_t base = *s_base_p;
    uint64_t* uk = a.out.ukeys + (int64_t)t * n;
    uint32_t* of = a.out.offs + (int64_t)t * (n + 1);
    if (agg == (uint32_t)len) {
        // every key distinct (the common case for fingerprints): bucket p = item p
        if (LSHB_OK((int64_t)base + len <= n))
            for (int p = u; p < len; p += kG2aT) {
                __stcs(uk + base + p, S.sk[p]);
                __stcs(of + base + p, (uint32_t)(lo + p));
            }
    } else {
        uint32_t b = base;
        for (int p0 = 0; p0 < len; p0 += kG2aT) {
            const int p = p0 + u;
            const uint64_t k = p < len ? S.sk[p] : 0ull;
            const bool h = p < len && (p == 0 || k != S.sk[p - 1]);
            uint32_t all;
            const uint32_t ex = cblock_excl_scan(h ? 1u : 0u, S.ws, &all);
            if (h && LSHB_OK((int64_t)b + ex < n)) {
                __stcs(uk + b + ex, k);
                __stcs(of + b + ex, (uint32_t)(lo + p));
            }
            b += all;
        }
    }
    if (bin == nb1 - 1 && u == 0) {
        a.out.nb[t] = base + agg;
        of[base + agg] = (uint32_t)n;
    }
}


__global__ void __launch_bounds__(kG2aT, LSHB_G2_CPS) g2a(G2Args a) {
    extern __shared__ __align__(16) unsigned char g2a_dsm[];
    G2aSmem& S = *reinterpret_cast<G2aSmem*>(g2a_dsm);
    __shared__ uint32_t s_tick, s_base;
    const int nb1 = a.nb1;
    const int64_t n = a.n;
    // bins are numbered through a dynamic ticket, so every bin this CTA looks back at
    // belongs to a CTA that is already running: the look-back cannot stall
    if (threadIdx.x == 0) s_tick = atomicAdd(a.ticket, 1u);
    {
        // g2_bin's shared state, zeroed under the ticket's latency
        uint4* c4 = reinterpret_cast<uint4*>(S.cnt);
        for (int w = threadIdx.x; w < kG2aCW / 4; w += kG2aT) c4[w] = make_uint4(0u, 0u, 0u, 0u);
        if (threadIdx.x == 0) {
            S.nlong = 0u;
            S.heads = 0u;
            S.nwl = 0u;
        }
    }
    cbar();
    // tables interleaved: the CTAs in flight cover ~1/L of every table's bins, so each
    // table's look-back chain only has to advance a few bins per CTA lifetime
    const int t = (int)(s_tick % (uint32_t)a.L), bin = (int)(s_tick / (uint32_t)a.L);
    // the fixed-capacity L1 layout's slots of this bin are loaded speculatively together
    // with the bin's bounds (one memory round trip instead of two); if the histogram
    // path produced the L1 output instead (*ovf != 0), the items are reloaded from it
    const int u = threadIdx.x;
    const int64_t fsrc = (int64_t)t * a.fix_tstride + (int64_t)bin * kG2aCap;
    uint64_t kr[kG2aIPT];
    uint32_t ir[kG2aIPT];
#pragma unroll
    for (int j = 0; j < kG2aIPT; ++j) {
        kr[j] = a.keys[fsrc + u + j * kG2aT];
        ir[j] = a.ids[fsrc + u + j * kG2aT];
    }
    const uint32_t* bs = a.binstart + (int64_t)t * (nb1 + 1);
    const int64_t lo = bs[bin];
    const int len = (int)((int64_t)bs[bin + 1] - lo);
    const bool fixed = a.ovf && *a.ovf == 0u;
    if (len > kG2aCap) {
        g2a_big_emit(a, t, bin, lo, len, &s_base);
        return;
    }
    if (!fixed) {
        const int64_t src = (int64_t)t * n + lo;
#pragma unroll
        for (int j = 0; j < kG2aIPT; ++j) {
            const int i = u + j * kG2aT;
            if (i < len) {
                kr[j] = a.keys[src + i];
                ir[j] = a.ids[src + i];
            }
        }
    }
    g2_bin(a, S, t, bin, lo, len, kr, ir, &s_base);
}

// Run-length encoding of fully sorted keys (LSD path): chunk c = items
// [c*kG2Cap, (c+1)*kG2Cap) of a table; heads by comparison with the previous item;
// bucket numbering by the same chained look-back as the per-chunk sort.
__global__ void __launch_bounds__(kG2Threads) g3_rle(const uint64_t* __restrict__ keys, int64_t n, int nchunks,
                                                     unsigned long long* __restrict__ state, IndexDev out) {
    __shared__ uint32_t ws[32];
    __shared__ uint32_t bc;
    constexpr int VP = kG2Cap / kG2Threads;
    const int t = blockIdx.x, c = blockIdx.y;
    const uint64_t* k = keys + (int64_t)t * n;
    const int64_t lo = (int64_t)c * kG2Cap;
    const int64_t r0 = lo + threadIdx.x * VP;
    uint64_t kv[VP];
    uint32_t hm = 0;
    uint64_t prev = (r0 > 0 && r0 <= n) ? k[r0 - 1] : 0ull;
#pragma unroll
    for (int j = 0; j < VP; ++j) {
        const int64_t r = r0 + j;
        kv[j] = r < n ? k[r] : 0ull;
        if (r < n && (r == 0 || kv[j] != prev)) hm |= 1u << j;
        prev = kv[j];
    }
    uint32_t utot;
    const uint32_t ex = block_excl_scan<kG2Threads>(__popc(hm), ws, &utot);
    if (threadIdx.x < 32) {
        const uint32_t pre = chained_prefix_warp(state + (int64_t)t * nchunks, c, utot);
        if (threadIdx.x == 0) bc = pre;
    }
    __syncthreads();
    const uint32_t base = bc;
    uint64_t* uk = out.ukeys + (int64_t)t * n;
    uint32_t* of = out.offs + (int64_t)t * (n + 1);
    uint32_t ub = base + ex;
#pragma unroll
    for (int j = 0; j < VP; ++j)
        if ((hm >> j) & 1u) {
            if (LSHB_OK(ub < (uint32_t)n)) {
                uk[ub] = kv[j];
                of[ub] = (uint32_t)(r0 + j);
            }
            ++ub;
        }
    if (threadIdx.x == 0 && c == nchunks - 1) {
        out.nb[t] = base + utot;
        of[base + utot] = (uint32_t)n;
    }
}

// big-bin path: per-warp 8-bit digit counts (16 KB), a run bitmap (1 KB) and its
// 8192 positions (16 KB)
static size_t g2_big_smem() { return 16384 + 1024 + 16384; }

size_t group_hist_words(int64_t n, int W) {
    return ((size_t)1 << group_l1_bits(n, W)) * group_tiles(n);
}
int group_bins(int64_t n, int W) { return 1 << group_l1_bits(n, W); }
int group_rle_chunks(int64_t n) { return (int)((n + kG2Cap - 1) / kG2Cap); }
size_t group_key_slots(int64_t n, int W) {
    if (n == 0 || group_is_lsd(W)) return (size_t)n;
    return std::max<size_t>((size_t)n, (size_t)group_bins(n, W) * kG2BinCap);
}
size_t group_spec_bytes() { return sizeof(L1Spec); }

static unsigned hist_grid(int T, int L, int num_sms) {
    return (unsigned)std::min<int64_t>((int64_t)T * L, (int64_t)num_sms * 8);
}

// One L1 counting pass (histogram, tile scan, bin starts, stable scatter) of every
// table by the digit of spec[0..L).
static cudaError_t l1_pass(const uint64_t* kin, const uint32_t* iin, uint64_t* kout, uint32_t* iout, int64_t n, int L,
                           const L1Spec* spec, int nb1, uint32_t id_base, GroupScratch& sc, uint32_t* biglist,
                           uint32_t* bigcount, int num_sms, cudaStream_t s, bool hist_done = false,
                           bool stable = true) {
    const int T = (int)group_tiles(n);
    if (!hist_done) {
        timing_begin("group_hist", s);
        g1_hist<<<hist_grid(T, L, num_sms), kG1Threads, nb1 * sizeof(uint32_t), s>>>(kin, n, const_cast<L1Spec*>(spec), nb1,
                                                                               sc.hist, T, 0, 64, 0, nullptr, nullptr, L);
        count_launch();
        timing_end("group_hist", s);
    }
    timing_begin("group_scan", s);
    const int64_t warps = (int64_t)L * ((nb1 + 31) / 32);
    g1_scan<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(sc.hist, T, L, nb1, sc.tot);
    count_launch();
    g1_binstart<<<L, 1024, 0, s>>>(sc.tot, nb1, n, sc.binstart, biglist, bigcount);
    count_launch();
    timing_end("group_scan", s);
    timing_begin("group_scatter", s);
    const bool ids = iin != nullptr;
    int nst = LSHB_SCATTER_NST;
    const size_t sm1 = g1_scatter_smem(nb1, stable || ids, nst);
    const int64_t items = (int64_t)T * L;
    const int grid = (int)std::min<int64_t>(items, (int64_t)num_sms * LSHB_SCATTER_CPS);
    cudaError_t e;
    if (!ids) {
        if (stable) {
            e = cudaFuncSetAttribute(g1_scatter<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
            if (e != cudaSuccess) return e;
            g1_scatter<true, true><<<grid, kSThreads, sm1, s>>>(kin, nullptr, kout, iout, n, spec, nb1, sc.hist,
                                                                sc.binstart, T, L, id_base, nst);
        } else {
            e = cudaFuncSetAttribute(g1_scatter<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
            if (e != cudaSuccess) return e;
            g1_scatter<true, false><<<grid, kSThreads, sm1, s>>>(kin, nullptr, kout, iout, n, spec, nb1, sc.hist,
                                                                 sc.binstart, T, L, id_base, nst);
        }
    } else {
        e = cudaFuncSetAttribute(g1_scatter<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
        if (e != cudaSuccess) return e;
        g1_scatter<false, true><<<grid, kSThreads, sm1, s>>>(kin, iin, kout, iout, n, spec, nb1, sc.hist, sc.binstart,
                                                             T, L, id_base, nst);
    }
    count_launch();
    timing_end("group_scatter", s);
    return cudaGetLastError();
}

cudaError_t launch_group(const uint64_t* keys, int64_t n, int L, uint32_t id_base, int W, GroupScratch& sc,
                         IndexDev& out, int* flags, cudaStream_t s) {
    // flags[1]: the handle's grouping-path hint (wide keys): > 0 after a build whose
    // fixed-capacity L1 pass overflowed (duplicate-heavy codes): the next builds go
    // straight to the histogram path, retrying the fixed one after 8 builds.  Only
    // the speed depends on it: both paths produce the same canonical index.
    uint32_t* hint = flags ? reinterpret_cast<uint32_t*>(flags + 1) : nullptr;
    cudaError_t e;
    if (n == 0) {
        e = cudaMemsetAsync(out.nb, 0, sizeof(uint32_t) * L, s);
        if (e != cudaSuccess) return e;
        return cudaMemsetAsync(out.offs, 0, sizeof(uint32_t) * L * (n + 1), s);
    }
    L1Spec* spec = reinterpret_cast<L1Spec*>(sc.spec);
    const bool lsd = group_is_lsd(W);
    const int B1 = group_l1_bits(n, W);
    const int nb1 = 1 << B1;
    timing_begin("group_hist", s);
    e = cudaMemsetAsync(sc.vmask, 0, sizeof(unsigned long long) * 2 * L, s);
    if (e != cudaSuccess) return e;
    const int T = (int)group_tiles(n);
    if (lsd) {
        g0_mask<<<dim3((unsigned)((n + 8191) / 8192), L), 256, 0, s>>>(keys, n, sc.vmask);
        count_launch();
        g0_spec<<<(L + 127) / 128, 128, 0, s>>>(sc.vmask, L, B1, 2, spec);
        count_launch();
    }
    timing_end("group_hist", s);
    if (lsd) {
        // narrow keys: full stable LSD sort on the varying bits (two passes), then RLE
        e = l1_pass(keys, nullptr, sc.keys_a, sc.ids_a, n, L, spec, nb1, id_base, sc, nullptr, nullptr, sc.num_sms, s);
        if (e != cudaSuccess) return e;
        uint64_t* kb = reinterpret_cast<uint64_t*>(sc.perm);
        e = l1_pass(sc.keys_a, sc.ids_a, kb, out.ids, n, L, spec + L, nb1, id_base, sc, nullptr, nullptr, sc.num_sms, s);
        if (e != cudaSuccess) return e;
        const int nch = (int)((n + kG2Cap - 1) / kG2Cap);
        timing_begin("group_sort", s);
        e = cudaMemsetAsync(sc.state, 0, sizeof(unsigned long long) * (size_t)L * nch, s);
        if (e != cudaSuccess) return e;
        g3_rle<<<dim3(L, nch), kG2Threads, 0, s>>>(kb, n, nch, sc.state, out);
        count_launch();
        timing_end("group_sort", s);
        return cudaGetLastError();
    }
    // wide keys.  (1) fixed-capacity L1 scatter on the top B1 bits with per-bin cursors
    // (no histogram pass, the keys are read once); (2) if a bin overflowed (skewed /
    // duplicate-heavy keys), the histogram path (varying-bit digit, per-tile counts,
    // stable bin starts, big-bin list) redoes the L1 pass — its kernels are gated on
    // the overflow word and exit at once otherwise.
    uint32_t* ovf = sc.bigcount + 2;
    e = cudaMemsetAsync(sc.bigcount, 0, 3 * sizeof(uint32_t), s);   // big-bin count, g2a ticket, overflow
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(sc.tot, 0, sizeof(uint32_t) * (size_t)L * nb1, s);   // bin cursors
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(sc.state, 0, sizeof(unsigned long long) * (size_t)L * nb1, s);   // look-back words
    if (e != cudaSuccess) return e;
    const int64_t fix_tstride = (int64_t)nb1 * kG2BinCap;
    {
        timing_begin("group_scatter", s);
        const int nst = LSHB_SCATTER_NST;
        const size_t smf = g1_scatter_smem(nb1, false, nst);
        e = cudaFuncSetAttribute(g1_scatter<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smf);
        if (e != cudaSuccess) return e;
        const int grid = (int)std::min<int64_t>((int64_t)T * L, (int64_t)sc.num_sms * LSHB_SCATTER_CPS);
        g1_scatter<true, false, true><<<grid, kSThreads, smf, s>>>(keys, nullptr, sc.keys_a, sc.ids_a, n, spec, nb1,
                                                                   sc.tot, sc.binstart, T, L, id_base, nst, nullptr,
                                                                   ovf, B1, W, fix_tstride, hint);
        count_launch();
        timing_end("group_scatter", s);
        timing_begin("group_scan", s);
        g1_fixscan<<<L, 1024, 0, s>>>(sc.tot, nb1, n, sc.binstart, spec, B1, W, ovf, hint);
        count_launch();
        timing_end("group_scan", s);
    }
    {
        // fallback (gated on *ovf)
        timing_begin("group_hist", s);
        g1_hist<<<hist_grid(T, L, sc.num_sms), kG1Threads, nb1 * sizeof(uint32_t), s>>>(keys, n, spec, nb1, sc.hist, T, 1,
                                                                                       W, B1, sc.vmask, ovf, L);
        count_launch();
        g0_spec<<<(L + 127) / 128, 128, 0, s>>>(sc.vmask, L, B1, 1, spec, ovf);
        count_launch();
        g1_hist<<<hist_grid(T, L, sc.num_sms), kG1Threads, nb1 * sizeof(uint32_t), s>>>(keys, n, spec, nb1, sc.hist, T, 2,
                                                                                       W, B1, nullptr, ovf, L);
        count_launch();
        timing_end("group_hist", s);
        timing_begin("group_scan", s);
        const int64_t warps = (int64_t)L * ((nb1 + 31) / 32);
        g1_scan<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(sc.hist, T, L, nb1, sc.tot, ovf);
        count_launch();
        g1_binstart<<<L, 1024, 0, s>>>(sc.tot, nb1, n, sc.binstart, sc.biglist, sc.bigcount, ovf);
        count_launch();
        timing_end("group_scan", s);
        timing_begin("group_scatter", s);
        const int nst = LSHB_SCATTER_NST;
        const size_t sm1 = g1_scatter_smem(nb1, false, nst);
        e = cudaFuncSetAttribute(g1_scatter<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
        if (e != cudaSuccess) return e;
        const int grid = (int)std::min<int64_t>((int64_t)T * L, (int64_t)sc.num_sms * LSHB_SCATTER_CPS);
        g1_scatter<true, false><<<grid, kSThreads, sm1, s>>>(keys, nullptr, sc.keys_a, sc.ids_a, n, spec, nb1, sc.hist,
                                                             sc.binstart, T, L, id_base, nst, ovf);
        count_launch();
        timing_end("group_scatter", s);
    }
    timing_begin("group_sort", s);
    G2Args a;
    a.keys = sc.keys_a;
    a.ids = sc.ids_a;
    a.binstart = sc.binstart;
    a.state = sc.state;
    a.scratch = sc.perm;
    a.spec = spec;
    a.n = n;
    a.L = L;
    a.nb1 = nb1;
    a.id_base = id_base;
    a.biglist = sc.biglist;
    a.bigcount = sc.bigcount;
    a.out = out;
    a.binheads = sc.tot;   // bin totals are dead after g1_binstart
    a.ticket = sc.bigcount + 1;
    a.ovf = ovf;
    a.fix_tstride = fix_tstride;
    const size_t smb = g2_big_smem();
    e = cudaFuncSetAttribute(g2_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(g2a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(G2aSmem));
    if (e != cudaSuccess) return e;
    const unsigned bins = (unsigned)((int64_t)L * nb1);
    g2_big<<<sc.num_sms, kG2Threads, smb, s>>>(a);   // bins larger than kG2aCap (usually none)
    count_launch();
    g2a<<<bins, kG2aT, sizeof(G2aSmem), s>>>(a);   // sort every bin; ids, ukeys, offs out
    count_launch();
    timing_end("group_sort", s);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K5: bucket lookup of query keys ("collect the index of all the
// elements ... hashed in hbar_t(q)").
// ---------------------------------------------------------------------------
// interp (64-bit fingerprint keys, uniform over [0, 2^64)): up to three rounds that
// interpolate the key's position between the current bounds and probe two positions
// a few standard deviations around it (independent loads: one memory round trip per
// round), then the binary search finishes.  Every probe only moves lo or hi past an
// index whose key is known to be < or >= the query key, so the result is the
// lower bound in every case (equal to the plain binary search), only the number of
// dependent loads changes (~9 instead of ~20 at 10^6 buckets).
__global__ void lookup_kernel(const uint64_t* __restrict__ qkeys, int64_t nq, int L, int64_t n, IndexDev idx,
                              int64_t* __restrict__ begin, int64_t* __restrict__ end, int interp) {
    const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= nq * L) return;
    const int64_t q = gi / L;
    const int t = (int)(gi % L);
    const uint64_t key = qkeys[(int64_t)t * nq + q];
    const uint64_t* uk = idx.ukeys + (int64_t)t * n;
    const uint32_t* of = idx.offs + (int64_t)t * (n + 1);
    const int64_t nb = idx.nb[t];
    // invariant: uk[i] < key for i < lo, uk[i] >= key for i >= hi; the keys in [lo, hi)
    // lie in [klo, khi]
    int64_t lo = 0, hi = nb;
    uint64_t klo = 0, khi = ~0ull;
    if (interp) {
#pragma unroll 1
        for (int r = 0; r < 3 && hi - lo > 64; ++r) {
            const double span = (double)(hi - lo);
            double phi = key <= klo ? 0.0 : key >= khi ? 1.0 : (double)(key - klo) / (double)(khi - klo);
            const int64_t g = lo + (int64_t)(phi * span);
            const int64_t dl = 2 + (int64_t)(2.0 * sqrt(span));
            const int64_t p1 = max(lo, g - dl), p2 = min(hi - 1, g + dl);
            const uint64_t v1 = uk[p1], v2 = uk[p2];
            if (v1 >= key) {
                hi = p1;
                khi = v1;
            } else {
                lo = p1 + 1;
                klo = v1;
                if (v2 >= key) {
                    hi = p2;
                    khi = v2;
                } else {
                    lo = p2 + 1;
                    klo = v2;
                }
            }
        }
    }
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (uk[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    int64_t b, e;
    if (lo < nb && uk[lo] == key) {
        b = of[lo];
        e = of[lo + 1];
    } else {
        b = e = of[lo];
    }
    begin[q * L + t] = b;
    end[q * L + t] = e;
}

cudaError_t launch_lookup(const uint64_t* qkeys, int64_t nq, int L, int64_t n, const IndexDev& idx, int64_t* begin,
                          int64_t* end, bool interp, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    const int64_t tot = nq * L;
    lookup_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(qkeys, nq, L, n, idx, begin, end, interp ? 1 : 0);
    return cudaGetLastError();
}

// Coarse counts from the sorted bucket keys: coarse bins are monotone in key order,
// so bin b of table t spans the buckets [lower_bound(b << s), lower_bound((b+1) << s))
// and its point count is a difference of two offsets (no atomics, deterministic).
__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* a, int64_t nb, uint64_t key) {
    int64_t lo = 0, hi = nb;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void counts_kernel(IndexDev idx, int64_t n, int L, int W, int B, uint32_t* counts) {
    const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nbins = (int64_t)1 << B;
    if (gi >= (int64_t)L * nbins) return;
    const int t = (int)(gi >> B);
    const uint64_t b = (uint64_t)(gi & (nbins - 1));
    const uint64_t* uk = idx.ukeys + (int64_t)t * n;
    const uint32_t* of = idx.offs + (int64_t)t * (n + 1);
    const int64_t nb = idx.nb[t];
    int64_t lo, hi;
    if (W > B) {
        const int sh = W - B;
        lo = lower_bound_u64(uk, nb, b << sh);
        hi = (b + 1 == (uint64_t)nbins) ? nb : lower_bound_u64(uk, nb, (b + 1) << sh);
    } else {
        lo = lower_bound_u64(uk, nb, b);
        hi = (lo < nb && uk[lo] == b) ? lo + 1 : lo;
    }
    counts[gi] = of[hi] - of[lo];
}

cudaError_t launch_counts(const IndexDev& idx, int64_t n, int L, int W, int B, uint32_t* counts, cudaStream_t s) {
    const int64_t tot = (int64_t)L << B;
    if (n == 0) return cudaMemsetAsync(counts, 0, sizeof(uint32_t) * tot, s);
    counts_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(idx, n, L, W, B, counts);
    return cudaGetLastError();
}

// Exclusive prefix of the all-gathered coarse counts (bin-major, rank-minor), one
// block per table: scan over bins of the totals, plus the counts of lower ranks.
__global__ void __launch_bounds__(1024) global_offsets_kernel(const uint32_t* __restrict__ all, int G, int rank, int L,
                                                             int B, int64_t* __restrict__ off) {
    __shared__ unsigned long long wsum[32];
    __shared__ unsigned long long carry_s;
    const int t = blockIdx.x;
    const int nb = 1 << B;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += 1024) {
        const int b = base + threadIdx.x;
        unsigned long long tot = 0, lower = 0;
        if (b < nb) {
            for (int r = 0; r < G; ++r) {
                const unsigned long long c = all[((int64_t)r * L + t) * nb + b];
                tot += c;
                if (r < rank) lower += c;
            }
        }
        unsigned long long x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            unsigned long long w = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            wsum[lane] = w;
        }
        __syncthreads();
        const unsigned long long excl = carry_s + (warp ? wsum[warp - 1] : 0ull) + x - tot;
        if (b < nb) off[(int64_t)t * nb + b] = (int64_t)(excl + lower);
        __syncthreads();
        if (threadIdx.x == 1023) carry_s = excl + tot;
        __syncthreads();
    }
}


cudaError_t launch_global_offsets(const uint32_t* all, int G, int rank, int L, int B, int64_t* off, cudaStream_t s) {
    global_offsets_kernel<<<L, 1024, 0, s>>>(all, G, rank, L, B, off);
    return cudaGetLastError();
}

// Cross-shard query runs: all_ranges int64 [G][2][M] = every rank's local (begin[M],
// end[M]) of the same M = nq*L (query, table) lookups.  The global bucket of (q, t) is
// the rank-order concatenation of the ranks' runs, so rank `rank`'s run starts at
// gbegin[j] = sum_{r < rank} (end_r[j] - begin_r[j]) inside it; gtotal[j] = its size.
__global__ void __launch_bounds__(256) query_runs_kernel(const int64_t* __restrict__ all, int G, int rank, int64_t M,
                                                          int64_t* __restrict__ gbegin, int64_t* __restrict__ gtotal) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
        int64_t lower = 0, tot = 0;
        for (int r = 0; r < G; ++r) {
            const int64_t sz = all[((int64_t)r * 2 + 1) * M + j] - all[(int64_t)r * 2 * M + j];
            tot += sz;
            if (r < rank) lower += sz;
        }
        gbegin[j] = lower;
        if (gtotal) gtotal[j] = tot;
    }
}

cudaError_t launch_query_runs(const int64_t* all, int G, int rank, int64_t M, int64_t* gbegin, int64_t* gtotal,
                              cudaStream_t s) {
    if (M == 0) return cudaSuccess;
    const int64_t blocks = (M + 255) / 256;
    query_runs_kernel<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, s>>>(all, G, rank, M, gbegin, gtotal);
    return cudaGetLastError();
}

}  // namespace lshb

