// group.cu — K3/K5: grouping points into the buckets of each of the L tables
// ("store every point p in bucket hbar_t(p)"; "arranging data
// points into several bins of hash tables based on their hashcode")
// and the bucket lookup of queries.  DESIGN.md §K3.
//
// Output order is canonical (reading B11): per table, ids sorted by (key, id),
// i.e. buckets by ascending unsigned key, ids ascending inside a bucket.
//
//   1. stable LSD counting-sort passes on the top 16 significant key bits
//      (8-bit digits; warp-level match_any ranking keeps each pass stable, so
//      ids stay ascending inside equal digits),
//   2. if keys are wider than 16 bits (E2LSH fingerprints, SRP with K > 16):
//      stable sort of each equal-top-16 segment by the full key (segments are
//      ~n/65536 long for fingerprints; long ones go to a CTA-level bitonic sort),
//   3. run-length encoding -> ukeys / offs / nb.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.hpp"

namespace lshb {

constexpr int kTile = 4096;        // items per radix tile
constexpr int kRT = 256;           // threads per radix block
constexpr int kRounds = kTile / kRT;
constexpr int kSegWin = 2048;      // positions owned by one segment-sort block
constexpr int kSegCap = 64;        // longest segment sorted by the windowed kernel (O(s^2) ranks)
constexpr int kSegBig = 8192;      // CTA bitonic capacity in shared memory

size_t group_tiles(int64_t n) { return (size_t)((n + kTile - 1) / kTile); }

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

template <bool IMPLICIT_IDS>
__global__ void __launch_bounds__(kRT) radix_upsweep(const uint64_t* __restrict__ keys, int64_t n, int sh,
                                                     uint32_t* __restrict__ hist, int T) {
    __shared__ uint32_t cnt[256];
    const int t = blockIdx.y, tile = blockIdx.x;
    cnt[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t* kt = keys + (int64_t)t * n;
    for (int r = 0; r < kRounds; ++r) {
        const int64_t i = (int64_t)tile * kTile + r * kRT + threadIdx.x;
        if (i < n) atomicAdd(&cnt[(kt[i] >> sh) & 255], 1u);
    }
    __syncthreads();
    hist[((int64_t)t * 256 + threadIdx.x) * T + tile] = cnt[threadIdx.x];
}

// Exclusive scan of `len` uint32 values per table (row stride `stride`) in place;
// writes the total to total_out[t] if non-null and also at a[len] if write_end.
__global__ void __launch_bounds__(1024) scan_rows(uint32_t* a, int64_t len, int64_t stride, uint32_t* total_out,
                                                  int write_end) {
    __shared__ uint32_t wsum[32];
    __shared__ uint32_t carry_s;
    uint32_t* row = a + (int64_t)blockIdx.x * stride;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int64_t base = 0; base < len; base += 1024) {
        const int64_t i = base + threadIdx.x;
        const uint32_t v = i < len ? row[i] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            wsum[lane] = w;
        }
        __syncthreads();
        const uint32_t carry = carry_s;
        const uint32_t excl = carry + (warp ? wsum[warp - 1] : 0u) + x - v;
        if (i < len) row[i] = excl;
        __syncthreads();
        if (threadIdx.x == 1023) carry_s = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (total_out) total_out[blockIdx.x] = carry_s;
        if (write_end) row[len] = carry_s;
    }
}

// Stable scatter of one 4096-item tile by an 8-bit digit.  Warp w owns the tile's
// items [512w, 512w+512) (coalesced 32-item rounds); a warp ranks its items with
// match_any against its own running per-digit counters (no block barrier per
// round), then one block-wide pass turns (digit, warp) counts into offsets.  Items
// are placed in digit order in shared memory and written out so that consecutive
// threads write consecutive addresses.  Order inside a digit = item order: stable.
template <bool IMPLICIT_IDS>
__global__ void __launch_bounds__(kRT) radix_downsweep(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ iin,
                                                       uint64_t* __restrict__ kout, uint32_t* __restrict__ iout,
                                                       int64_t n, int sh, const uint32_t* __restrict__ hist, int T,
                                                       uint32_t id_base) {
    constexpr int W = kRT / 32;             // warps
    constexpr int PER_WARP = kTile / W;     // 512 items
    constexpr int R = PER_WARP / 32;        // 16 rounds
    __shared__ uint32_t wrun[W][256];       // per-warp running digit counts, then warp offsets
    __shared__ uint32_t tile_off[256];
    __shared__ uint32_t local_off[256];
    __shared__ uint32_t ws[W];
    extern __shared__ __align__(16) unsigned char dsm[];
    uint64_t* sk = reinterpret_cast<uint64_t*>(dsm);                  // [kTile]
    uint32_t* si = reinterpret_cast<uint32_t*>(dsm + kTile * 8);      // [kTile]
    const int t = blockIdx.y, tile = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int w = 0; w < W; ++w) wrun[w][threadIdx.x] = 0;
    tile_off[threadIdx.x] = hist[((int64_t)t * 256 + threadIdx.x) * T + tile];
    __syncthreads();
    const int64_t tb = (int64_t)t * n;
    const int64_t base = (int64_t)tile * kTile + warp * PER_WARP;
    uint64_t key[R];
    uint32_t id[R], slot[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = base + r * 32 + lane;
        const bool valid = i < n;
        key[r] = valid ? kin[tb + i] : ~0ull;
        id[r] = valid ? (IMPLICIT_IDS ? id_base + (uint32_t)i : iin[tb + i]) : 0u;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = base + r * 32 + lane;
        const bool valid = i < n;
        const uint32_t dg = valid ? ((uint32_t)(key[r] >> sh) & 255u) : 256u;
        const uint32_t peers = __match_any_sync(0xffffffffu, dg);
        const uint32_t rank = __popc(peers & lanemask_lt());
        uint32_t before = 0;
        if (valid) before = wrun[warp][dg];
        __syncwarp();
        if (valid && rank == 0) wrun[warp][dg] = before + __popc(peers);
        __syncwarp();
        slot[r] = valid ? (dg << 16) | (before + rank) : 0xffffffffu;
    }
    __syncthreads();
    {   // per digit: exclusive prefix over warps, and the tile's digit totals
        const int dd = threadIdx.x;
        uint32_t acc = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint32_t c = wrun[w][dd];
            wrun[w][dd] = acc;
            acc += c;
        }
        // exclusive scan of totals across digits -> local_off
        uint32_t x = acc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) ws[warp] = x;
        __syncthreads();
        uint32_t pre = 0;
        for (int w = 0; w < warp; ++w) pre += ws[w];
        local_off[dd] = pre + x - acc;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (slot[r] != 0xffffffffu) {
            const uint32_t dg = slot[r] >> 16;
            const uint32_t p = local_off[dg] + wrun[warp][dg] + (slot[r] & 0xffffu);
            sk[p] = key[r];
            si[p] = id[r];
        }
    }
    __syncthreads();
    const int64_t cnt = min((int64_t)kTile, n - (int64_t)tile * kTile);
    for (int p = threadIdx.x; p < cnt; p += kRT) {
        const uint64_t k = sk[p];
        const uint32_t dg = (uint32_t)(k >> sh) & 255u;
        const uint32_t pos = tile_off[dg] + (p - local_off[dg]);
        kout[tb + pos] = k;
        iout[tb + pos] = si[p];
    }
}

__device__ __forceinline__ bool kless(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// Segments of equal top-16 significant bits: stable sort by the full key.  One
// block owns the segments whose head lies in its window of kSegWin positions and
// loads the window plus kSegCap positions of look-ahead into shared memory.
// Segment heads are found with one block scan; each item's rank inside its
// segment is #{smaller keys} + #{equal keys before it} (items arrive id-ascending
// inside a segment, so this is the stable order).  Longer segments go to the
// overflow list (segsort_big).
__global__ void __launch_bounds__(256) segsort_window(uint64_t* __restrict__ keys, uint32_t* __restrict__ ids, int64_t n,
                                                      int pre_sh, uint32_t* overflow, int cap) {
    constexpr int LEN = kSegWin + kSegCap;
    constexpr int PER = (LEN + 255) / 256;
    __shared__ uint64_t sk[LEN];
    __shared__ uint32_t si[LEN];
    __shared__ uint16_t seg_of[LEN];
    __shared__ uint16_t seg_start[LEN + 1];
    __shared__ uint32_t ws[8];
    __shared__ int nseg_s;
    const int t = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t w0 = (int64_t)blockIdx.x * kSegWin;
    uint64_t* k = keys + (int64_t)t * n;
    uint32_t* d = ids + (int64_t)t * n;
    const int len = (int)min((int64_t)LEN, n - w0);
    const int own = (int)min((int64_t)kSegWin, n - w0);
    for (int a = threadIdx.x; a < len; a += blockDim.x) {
        sk[a] = k[w0 + a];
        si[a] = d[w0 + a];
    }
    const uint64_t prev_pre = w0 > 0 ? (k[w0 - 1] >> pre_sh) : ~0ull;
    __syncthreads();
    // head flags over my PER consecutive positions, block scan -> segment ids
    const int a0 = threadIdx.x * PER;
    uint32_t flags = 0, cntf = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int a = a0 + q;
        if (a < len) {
            const uint64_t pr = a == 0 ? prev_pre : (sk[a - 1] >> pre_sh);
            if ((sk[a] >> pre_sh) != pr) {
                flags |= 1u << q;
                ++cntf;
            }
        }
    }
    uint32_t x = cntf;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    uint32_t sid = 0;
    for (int w = 0; w < warp; ++w) sid += ws[w];
    sid += x - cntf;  // heads before my first position
    if (threadIdx.x == 255) nseg_s = (int)(sid + cntf);
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int a = a0 + q;
        if (a < len) {
            if (flags >> q & 1u) {
                seg_start[sid] = (uint16_t)a;
                ++sid;
            }
            seg_of[a] = (uint16_t)(sid == 0 ? 0xffffu : sid - 1);  // 0xffff: previous window's segment
        }
    }
    __syncthreads();
    const int nseg = nseg_s;
    for (int li = threadIdx.x; li < len; li += blockDim.x) {
        const uint32_t sg = seg_of[li];
        if (sg == 0xffffu) continue;
        const int h = seg_start[sg];
        if (h >= own) continue;                              // head in the next window
        const int e = (int)sg + 1 < nseg ? seg_start[sg + 1] : len;
        const uint64_t pre = sk[li] >> pre_sh;
        const bool beyond = (e == len) && (w0 + len < n) && (k[w0 + len] >> pre_sh) == pre;
        if (beyond || e - h > kSegCap) {
            if (li == h) {                                   // the head reports the long segment once
                // end of the prefix run: keys are sorted by prefix, so binary search
                int64_t a = w0 + e, b = n;
                while (a < b) {
                    const int64_t mid = (a + b) >> 1;
                    if ((k[mid] >> pre_sh) == pre) a = mid + 1;
                    else b = mid;
                }
                const int64_t ge = a;
                const uint32_t slot = atomicAdd(overflow, 1u);
                if ((int)slot < cap) {
                    overflow[1 + 3 * slot] = (uint32_t)t;
                    overflow[2 + 3 * slot] = (uint32_t)(w0 + h);
                    overflow[3 + 3 * slot] = (uint32_t)ge;
                }
            }
            continue;
        }
        if (e - h == 1) continue;
        const uint64_t kv = sk[li];
        int rank = 0;
        for (int j = h; j < e; ++j) {
            const uint64_t kj = sk[j];
            rank += (kj < kv || (kj == kv && j < li)) ? 1 : 0;
        }
        k[w0 + h + rank] = kv;
        d[w0 + h + rank] = si[li];
    }
}

// Sorting network with ascending comparators only (bitonic sort with a "flip" first
// merge step), so indices >= len behave as +infinity and need no padding.
template <typename KeyAt, typename Swap>
__device__ void ascending_network(int64_t len, KeyAt less_at, Swap swap_at, bool smem) {
    int64_t P = 1;
    while (P < len) P <<= 1;
    for (int64_t size = 2; size <= P; size <<= 1) {
        for (int64_t stride = size >> 1; stride > 0; stride >>= 1) {
            const bool flip = (stride == (size >> 1));
            for (int64_t i = threadIdx.x; i < (P >> 1); i += blockDim.x) {
                int64_t a, b;
                if (flip) {
                    const int64_t blk = i / stride, j = i % stride;
                    a = blk * size + j;
                    b = blk * size + size - 1 - j;
                } else {
                    a = (i / stride) * 2 * stride + (i % stride);
                    b = a + stride;
                }
                if (b < len && less_at(b, a)) swap_at(a, b);
            }
            if (smem) __syncthreads();
            else {
                __threadfence_block();
                __syncthreads();
            }
        }
    }
}

// Long equal-prefix segment (many equal keys, e.g. duplicate points or empty codes):
// one CTA runs a stable LSD radix sort of the segment on the key bits below the
// common prefix (8-bit digits, digits that are constant over the segment are
// skipped), ping-ponging with the free scratch buffers.  Items arrive id-ascending
// and every pass is stable, so the result is the (key, id) order.
__device__ void cta_radix_segment(uint64_t* k, uint32_t* d, uint64_t* k2, uint32_t* d2, int64_t len, int low_bits,
                                  uint32_t* s_cnt, uint32_t* s_wcnt, uint32_t* s_woff, uint64_t* s_red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // which digits vary across the segment?
    uint64_t orv = 0, andv = ~0ull;
    for (int64_t a = threadIdx.x; a < len; a += blockDim.x) {
        orv |= k[a];
        andv &= k[a];
    }
    for (int o = 16; o > 0; o >>= 1) {
        orv |= __shfl_xor_sync(0xffffffffu, orv, o);
        andv &= __shfl_xor_sync(0xffffffffu, andv, o);
    }
    if (lane == 0) {
        s_red[2 * warp] = orv;
        s_red[2 * warp + 1] = andv;
    }
    __syncthreads();
    orv = 0;
    andv = ~0ull;
    for (int w = 0; w < nw; ++w) {
        orv |= s_red[2 * w];
        andv &= s_red[2 * w + 1];
    }
    const uint64_t varying = orv ^ andv;
    __syncthreads();
    uint64_t *src_k = k, *dst_k = k2;
    uint32_t *src_d = d, *dst_d = d2;
    for (int sh = 0; sh < low_bits; sh += 8) {
        if (((varying >> sh) & 255u) == 0) continue;
        // histogram
        for (int i = threadIdx.x; i < 256; i += blockDim.x) s_cnt[i] = 0;
        __syncthreads();
        for (int64_t a = threadIdx.x; a < len; a += blockDim.x) atomicAdd(&s_cnt[(src_k[a] >> sh) & 255u], 1u);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t acc = 0;
            for (int i = 0; i < 256; ++i) {
                const uint32_t c = s_cnt[i];
                s_cnt[i] = acc;
                acc += c;
            }
        }
        __syncthreads();
        // stable scatter in rounds of blockDim items
        for (int64_t base = 0; base < len; base += blockDim.x) {
            const int64_t a = base + threadIdx.x;
            const bool valid = a < len;
            const uint64_t key = valid ? src_k[a] : 0;
            const uint32_t id = valid ? src_d[a] : 0;
            const uint32_t dg = valid ? (uint32_t)(key >> sh) & 255u : 256u;
            const uint32_t peers = __match_any_sync(0xffffffffu, dg);
            const uint32_t rank = __popc(peers & lanemask_lt());
            for (int i = threadIdx.x; i < nw * 256; i += blockDim.x) s_wcnt[i] = 0;
            __syncthreads();
            if (valid && rank == 0) s_wcnt[warp * 256 + dg] = __popc(peers);
            __syncthreads();
            for (int dd = threadIdx.x; dd < 256; dd += blockDim.x) {
                uint32_t acc = s_cnt[dd];
                for (int w = 0; w < nw; ++w) {
                    s_woff[w * 256 + dd] = acc;
                    acc += s_wcnt[w * 256 + dd];
                }
                s_cnt[dd] = acc;
            }
            __syncthreads();
            if (valid) {
                const uint32_t pos = s_woff[warp * 256 + dg] + rank;
                dst_k[pos] = key;
                dst_d[pos] = id;
            }
            __syncthreads();
        }
        uint64_t* tk = src_k;
        src_k = dst_k;
        dst_k = tk;
        uint32_t* td = src_d;
        src_d = dst_d;
        dst_d = td;
        __threadfence_block();
        __syncthreads();
    }
    if (src_k != k) {  // odd number of passes: copy back
        for (int64_t a = threadIdx.x; a < len; a += blockDim.x) {
            k[a] = src_k[a];
            d[a] = src_d[a];
        }
    }
}

__global__ void __launch_bounds__(1024) segsort_big(uint64_t* __restrict__ keys, uint32_t* __restrict__ ids,
                                                    uint64_t* __restrict__ scratch_k, uint32_t* __restrict__ scratch_d,
                                                    int64_t n, int low_bits, const uint32_t* overflow, int cap,
                                                    int* flags) {
    extern __shared__ __align__(16) unsigned char sm[];
    uint64_t* sk = reinterpret_cast<uint64_t*>(sm);
    uint32_t* si = reinterpret_cast<uint32_t*>(sm + kSegBig * sizeof(uint64_t));
    __shared__ uint32_t s_cnt[256];
    __shared__ uint64_t s_red[64];
    const uint32_t count = min(overflow[0], (uint32_t)cap);
    if (blockIdx.x == 0 && threadIdx.x == 0 && overflow[0] > (uint32_t)cap) atomicOr(flags, 4);
    for (uint32_t e = blockIdx.x; e < count; e += gridDim.x) {
        const int t = overflow[1 + 3 * e];
        const int64_t lo = overflow[2 + 3 * e], hi = overflow[3 + 3 * e];
        uint64_t* k = keys + (int64_t)t * n + lo;
        uint32_t* d = ids + (int64_t)t * n + lo;
        const int64_t len = hi - lo;
        {   // all keys equal (repeated code tuples): already in id order
            __shared__ int s_neq;
            if (threadIdx.x == 0) s_neq = 0;
            __syncthreads();
            const uint64_t k0 = k[0];
            int neq = 0;
            for (int64_t a = threadIdx.x; a < len && !neq; a += blockDim.x) neq = k[a] != k0;
            if (neq) s_neq = 1;
            __syncthreads();
            const int any = s_neq;
            __syncthreads();
            if (!any) continue;
        }
        // the per-warp count tables live in the dynamic smem area (unused by the partition)
        uint32_t* s_wcnt = reinterpret_cast<uint32_t*>(sm);
        uint32_t* s_woff = s_wcnt + 32 * 256;
        uint64_t* k2 = scratch_k + (int64_t)t * n + lo;
        uint32_t* d2 = scratch_d + (int64_t)t * n + lo;
        // Long segments are dominated by repeated keys (duplicate points, empty codes):
        // stable 3-way partition around the middle item's key first; the "equal" part is
        // already in id order, only the rest needs sorting.
        const uint64_t pivot = k[len / 2];
        __shared__ uint32_t s_lt, s_eq;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        if (threadIdx.x == 0) {
            s_lt = 0;
            s_eq = 0;
        }
        __syncthreads();
        {
            uint32_t lt = 0, eq = 0;
            for (int64_t a = threadIdx.x; a < len; a += blockDim.x) {
                lt += k[a] < pivot;
                eq += k[a] == pivot;
            }
            atomicAdd(&s_lt, lt);
            atomicAdd(&s_eq, eq);
        }
        __syncthreads();
        const uint32_t nlt = s_lt, neq = s_eq;
        uint32_t base0 = 0, base1 = nlt, base2 = nlt + neq;
        for (int64_t b0 = 0; b0 < len; b0 += blockDim.x) {
            const int64_t a = b0 + threadIdx.x;
            const bool valid = a < len;
            const uint64_t key = valid ? k[a] : 0;
            const uint32_t cls = !valid ? 3u : (key < pivot ? 0u : (key == pivot ? 1u : 2u));
            const uint32_t m0 = __ballot_sync(0xffffffffu, cls == 0), m1 = __ballot_sync(0xffffffffu, cls == 1),
                           m2 = __ballot_sync(0xffffffffu, cls == 2);
            if (lane == 0) {
                s_wcnt[warp * 3 + 0] = __popc(m0);
                s_wcnt[warp * 3 + 1] = __popc(m1);
                s_wcnt[warp * 3 + 2] = __popc(m2);
            }
            __syncthreads();
            uint32_t pre0 = base0, pre1 = base1, pre2 = base2;
            for (int w = 0; w < warp; ++w) {
                pre0 += s_wcnt[w * 3];
                pre1 += s_wcnt[w * 3 + 1];
                pre2 += s_wcnt[w * 3 + 2];
            }
            const uint32_t lm = (1u << lane) - 1u;
            if (valid) {
                const uint32_t pos = cls == 0 ? pre0 + __popc(m0 & lm) : cls == 1 ? pre1 + __popc(m1 & lm)
                                                                                  : pre2 + __popc(m2 & lm);
                k2[pos] = key;
                d2[pos] = d[a];
            }
            for (int w = 0; w < nw; ++w) {
                base0 += s_wcnt[w * 3];
                base1 += s_wcnt[w * 3 + 1];
                base2 += s_wcnt[w * 3 + 2];
            }
            __syncthreads();
        }
        __threadfence_block();
        __syncthreads();
        for (int64_t a = threadIdx.x; a < len; a += blockDim.x) {
            k[a] = k2[a];
            d[a] = d2[a];
        }
        __threadfence_block();
        __syncthreads();
        const int64_t ngt = len - nlt - neq;
        const int64_t part_lo[2] = {0, (int64_t)nlt + neq};
        const int64_t part_len[2] = {(int64_t)nlt, ngt};
        for (int q = 0; q < 2; ++q) {
            const int64_t plen = part_len[q];
            if (plen <= 1) continue;
            uint64_t* pk = k + part_lo[q];
            uint32_t* pd = d + part_lo[q];
            if (plen <= kSegBig) {
                for (int64_t a = threadIdx.x; a < plen; a += blockDim.x) {
                    sk[a] = pk[a];
                    si[a] = pd[a];
                }
                __syncthreads();
                ascending_network(
                    plen, [&](int64_t x, int64_t y) { return kless(sk[x], si[x], sk[y], si[y]); },
                    [&](int64_t x, int64_t y) {
                        const uint64_t tk = sk[x]; sk[x] = sk[y]; sk[y] = tk;
                        const uint32_t ti = si[x]; si[x] = si[y]; si[y] = ti;
                    },
                    true);
                for (int64_t a = threadIdx.x; a < plen; a += blockDim.x) {
                    pk[a] = sk[a];
                    pd[a] = si[a];
                }
                __syncthreads();
            } else {
                cta_radix_segment(pk, pd, k2 + part_lo[q], d2 + part_lo[q], plen, low_bits, s_cnt, s_wcnt, s_woff,
                                  s_red);
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kRT) rle_count(const uint64_t* __restrict__ keys, int64_t n, uint32_t* tile_aux,
                                                 int T) {
    __shared__ uint32_t c;
    const int t = blockIdx.y, tile = blockIdx.x;
    if (threadIdx.x == 0) c = 0;
    __syncthreads();
    const uint64_t* k = keys + (int64_t)t * n;
    uint32_t local = 0;
    for (int r = 0; r < kRounds; ++r) {
        const int64_t i = (int64_t)tile * kTile + r * kRT + threadIdx.x;
        if (i < n && (i == 0 || k[i] != k[i - 1])) ++local;
    }
    atomicAdd(&c, local);
    __syncthreads();
    if (threadIdx.x == 0) tile_aux[(int64_t)t * (T + 1) + tile] = c;
}

__global__ void __launch_bounds__(kRT) rle_write(const uint64_t* __restrict__ keys, int64_t n,
                                                 const uint32_t* tile_aux, int T, IndexDev out) {
    __shared__ uint32_t wsum[kRT / 32];
    __shared__ uint32_t base_s;
    const int t = blockIdx.y, tile = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t* k = keys + (int64_t)t * n;
    if (threadIdx.x == 0) base_s = tile_aux[(int64_t)t * (T + 1) + tile];
    __syncthreads();
    for (int r = 0; r < kRounds; ++r) {
        const int64_t i = (int64_t)tile * kTile + r * kRT + threadIdx.x;
        const bool head = i < n && (i == 0 || k[i] != k[i - 1]);
        const uint32_t ball = __ballot_sync(0xffffffffu, head);
        if (lane == 0) wsum[warp] = __popc(ball);
        __syncthreads();
        uint32_t before = base_s;
        for (int w = 0; w < warp; ++w) before += wsum[w];
        if (head) {
            const uint32_t b = before + __popc(ball & lanemask_lt());
            out.ukeys[(int64_t)t * n + b] = k[i];
            out.offs[(int64_t)t * (n + 1) + b] = (uint32_t)i;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t s = 0;
            for (int w = 0; w < kRT / 32; ++w) s += wsum[w];
            base_s += s;
        }
        __syncthreads();
    }
}

__global__ void rle_finish(IndexDev out, const uint32_t* tile_aux, int T, int64_t n, int L) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= L) return;
    const uint32_t nb = tile_aux[(int64_t)t * (T + 1) + T];
    out.nb[t] = nb;
    out.offs[(int64_t)t * (n + 1) + nb] = (uint32_t)n;
}

cudaError_t launch_group(const uint64_t* keys, int64_t n, int L, uint32_t id_base, int W, GroupScratch& sc,
                         IndexDev& out, int* flags, cudaStream_t s) {
    cudaError_t e;
    if (n == 0) {
        e = cudaMemsetAsync(out.nb, 0, sizeof(uint32_t) * L, s);
        if (e != cudaSuccess) return e;
        return cudaMemsetAsync(out.offs, 0, sizeof(uint32_t) * L * (n + 1), s);
    }
    const int T = (int)group_tiles(n);
    const dim3 g2(T, L);
    // digit shifts covering the top 16 significant bits, low digit first
    int shifts[2];
    int npass;
    if (W <= 8) {
        shifts[0] = 0;
        npass = 1;
    } else if (W <= 16) {
        shifts[0] = 0;
        shifts[1] = 8;
        npass = 2;
    } else {
        shifts[0] = W - 16;
        shifts[1] = W - 8;
        npass = 2;
    }
    // pass outputs alternate keys_a, keys_b (keys_b may alias the input keys:
    // the input is fully consumed by pass 0, which writes keys_a)
    const uint64_t* kin = keys;
    const uint32_t* iin = nullptr;
    for (int p = 0; p < npass; ++p) {
        const bool lastp = (p == npass - 1);
        uint64_t* kout = (p == 0) ? sc.keys_a : sc.keys_b;
        uint32_t* iout = lastp ? out.ids : sc.ids_a;
        timing_begin("radix_upsweep", s);
        if (p == 0) radix_upsweep<true><<<g2, kRT, 0, s>>>(kin, n, shifts[p], sc.hist, T);
        else radix_upsweep<false><<<g2, kRT, 0, s>>>(kin, n, shifts[p], sc.hist, T);
        count_launch();
        timing_end("radix_upsweep", s);
        timing_begin("radix_scan", s);
        scan_rows<<<L, 1024, 0, s>>>(sc.hist, (int64_t)256 * T, (int64_t)256 * T, nullptr, 0);
        count_launch();
        timing_end("radix_scan", s);
        timing_begin("radix_downsweep", s);
        const int dsm = kTile * 12;
        if (p == 0) {
            cudaFuncSetAttribute(radix_downsweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dsm);
            radix_downsweep<true><<<g2, kRT, dsm, s>>>(kin, iin, kout, iout, n, shifts[p], sc.hist, T, id_base);
        } else {
            cudaFuncSetAttribute(radix_downsweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dsm);
            radix_downsweep<false><<<g2, kRT, dsm, s>>>(kin, iin, kout, iout, n, shifts[p], sc.hist, T, id_base);
        }
        count_launch();
        timing_end("radix_downsweep", s);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        kin = kout;
        iin = iout;
    }
    uint64_t* sorted = (npass == 1) ? sc.keys_a : sc.keys_b;
    if (W > 16) {
        timing_begin("segsort", s);
        e = cudaMemsetAsync(sc.overflow, 0, sizeof(uint32_t), s);
        if (e != cudaSuccess) return e;
        const dim3 gw((unsigned)((n + kSegWin - 1) / kSegWin), L);
        segsort_window<<<gw, 256, 0, s>>>(sorted, out.ids, n, W - 16, sc.overflow, sc.overflow_cap);
        count_launch();
        timing_end("segsort", s);
        timing_begin("segsort_long", s);
        const size_t smem = kSegBig * (sizeof(uint64_t) + sizeof(uint32_t));
        cudaFuncSetAttribute(segsort_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        // scratch for long segments: the pass-0 buffers are free once pass 1 has run
        segsort_big<<<148, 1024, smem, s>>>(sorted, out.ids, sc.keys_a, sc.ids_a, n, W - 16, sc.overflow,
                                            sc.overflow_cap, flags);
        count_launch();
        timing_end("segsort_long", s);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    timing_begin("rle", s);
    rle_count<<<g2, kRT, 0, s>>>(sorted, n, sc.tile_aux, T);
    count_launch();
    scan_rows<<<L, 1024, 0, s>>>(sc.tile_aux, T, T + 1, nullptr, 1);
    count_launch();
    rle_write<<<g2, kRT, 0, s>>>(sorted, n, sc.tile_aux, T, out);
    count_launch();
    rle_finish<<<(L + 127) / 128, 128, 0, s>>>(out, sc.tile_aux, T, n, L);
    count_launch();
    timing_end("rle", s);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K5: bucket lookup of query keys ("collect the index of all the
// elements ... hashed in hbar_t(q)").
// ---------------------------------------------------------------------------
__global__ void lookup_kernel(const uint64_t* __restrict__ qkeys, int64_t nq, int L, int64_t n, IndexDev idx,
                              int64_t* __restrict__ begin, int64_t* __restrict__ end) {
    const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= nq * L) return;
    const int64_t q = gi / L;
    const int t = (int)(gi % L);
    const uint64_t key = qkeys[(int64_t)t * nq + q];
    const uint64_t* uk = idx.ukeys + (int64_t)t * n;
    const uint32_t* of = idx.offs + (int64_t)t * (n + 1);
    int64_t lo = 0, hi = idx.nb[t];
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (uk[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    int64_t b, e;
    if (lo < idx.nb[t] && uk[lo] == key) {
        b = of[lo];
        e = of[lo + 1];
    } else {
        b = e = of[lo];
    }
    begin[q * L + t] = b;
    end[q * L + t] = e;
}

cudaError_t launch_lookup(const uint64_t* qkeys, int64_t nq, int L, int64_t n, const IndexDev& idx, int64_t* begin,
                          int64_t* end, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    const int64_t tot = nq * L;
    lookup_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(qkeys, nq, L, n, idx, begin, end);
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

}  // namespace lshb

