// knn.cu — query completion: for each query, the union of its
// L buckets ("collect the index of all the elements ... hashed in hbar_t(q)",
// PAPER.md:155), exact re-rank and top-k under the family's similarity (§6
// Euclidean distance for the E2LSH family, cosine similarity
// for the SRP family).  Readings C1/C2: bucket entries in table order,
// capped at max_cand entries before removing duplicates; squared L2 ascending or
// cosine descending (0 when a norm is 0), ties by ascending id.
//
// One CTA per query: candidate ids gathered from the L bucket ranges into shared
// memory, bitonic-sorted and deduplicated; one warp per candidate computes the
// exact score with 128-bit loads of the base row; (orderable score, id) keys are
// bitonic-sorted and the first k written.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.hpp"

namespace lshb {

namespace {
constexpr int kQT = 1024;   // 32 warps score candidates in parallel
constexpr int kQW = kQT / 32;

__device__ __forceinline__ uint32_t ord_f32(float f) {   // ascending float -> ascending uint
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

template <typename T>
__device__ void bitonic_sort(T* v, int P) {   // ascending, P a power of two, whole block
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < (P >> 1); i += kQT) {
                const int lo = 2 * stride * (i / stride) + (i % stride), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const T a = v[lo], b = v[hi];
                if ((a > b) == up) {
                    v[lo] = b;
                    v[hi] = a;
                }
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ uint32_t block_excl(uint32_t x, uint32_t* ws, uint32_t* tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) ws[warp] = v;
    __syncthreads();
    uint32_t pre = 0, all = 0;
    for (int w = 0; w < kQW; ++w) {
        if (w < warp) pre += ws[w];
        all += ws[w];
    }
    __syncthreads();
    if (tot) *tot = all;
    return pre + v - x;
}
}  // namespace

struct KnnArgs {
    IndexDev idx;
    int64_t n;
    int L;
    uint32_t id_base;
    const int64_t* begin;   // [nq][L]
    const int64_t* end;
    const float* X;         // base rows, row = id - id_base
    int64_t ldx;
    int d;
    const float* Q;
    int64_t ldq;
    int k, max_cand, cosine, vec;
    int64_t* out_ids;       // [nq][k]
    float* out_score;       // [nq][k]
    int32_t* out_ncand;     // [nq]
};

__global__ void __launch_bounds__(kQT) knn_kernel(KnnArgs a, int P) {
    extern __shared__ __align__(16) unsigned char dsm[];
    unsigned long long* key = reinterpret_cast<unsigned long long*>(dsm);   // [P]
    uint32_t* cand = reinterpret_cast<uint32_t*>(key + P);                  // [P]
    uint32_t* pref = cand + P;                                              // [L+1]
    __shared__ uint32_t ws[kQW];
    __shared__ uint32_t s_u;
    __shared__ float s_qn;
    const int64_t qi = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int L = a.L;
    // 1. bucket sizes of the L tables, prefix in table order.  Only the first max_cand
    //    entries are used, so sizes and the prefix saturate at max_cand (no u32 wrap;
    //    the saturated prefix stays non-decreasing for the search below)
    const uint32_t cap = (uint32_t)a.max_cand;
    uint32_t carry = 0;
    for (int t0 = 0; t0 < L; t0 += kQT) {
        const int t = t0 + threadIdx.x;
        const int64_t sz = t < L ? a.end[qi * L + t] - a.begin[qi * L + t] : 0;
        const uint32_t c = (uint32_t)(sz < (int64_t)cap ? sz : (int64_t)cap);
        uint32_t tot;
        const uint32_t ex = block_excl(c, ws, &tot);   // <= kQT * cap < 2^32
        if (t < L) pref[t] = min(cap, carry + ex);
        carry = min(cap, carry + tot);
    }
    if (threadIdx.x == 0) pref[L] = carry;
    __syncthreads();
    const int total = (int)min((uint32_t)a.max_cand, pref[L]);
    // 2. gather candidate ids (table order, capped)
    for (int i = threadIdx.x; i < P; i += kQT) {
        uint32_t v = 0xffffffffu;
        if (i < total) {
            int lo = 0, hi = L;   // last t with pref[t] <= i
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (pref[mid] <= (uint32_t)i) lo = mid;
                else hi = mid;
            }
            v = a.idx.ids[(int64_t)lo * a.n + a.begin[qi * L + lo] + (i - pref[lo])];
        }
        cand[i] = v;
    }
    __syncthreads();
    // 3. sort + dedup (distinct ids -> key[] as u32 scratch, then back)
    bitonic_sort(cand, P);
    uint32_t* uniq = reinterpret_cast<uint32_t*>(key);
    uint32_t ub = 0;
    for (int i0 = 0; i0 < P; i0 += kQT) {
        const int i = i0 + threadIdx.x;
        const bool head = i < P && cand[i] != 0xffffffffu && (i == 0 || cand[i] != cand[i - 1]);
        uint32_t tot;
        const uint32_t ex = block_excl(head ? 1u : 0u, ws, &tot);
        if (head) uniq[ub + ex] = cand[i];
        ub += tot;
    }
    __syncthreads();
    const int u = (int)ub;
    for (int i = threadIdx.x; i < u; i += kQT) cand[i] = uniq[i];
    if (threadIdx.x == 0) s_u = ub;
    // query norm (cosine)
    if (warp == 0) {
        const float* q = a.Q + qi * a.ldq;
        float s = 0.f;
        for (int c = lane; c < a.d; c += 32) s = fmaf(q[c], q[c], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) s_qn = sqrtf(s);
    }
    __syncthreads();
    // 4. exact scores, one warp per candidate
    const float* q = a.Q + qi * a.ldq;
    for (int j = warp; j < u; j += kQW) {
        const uint32_t id = cand[j];
        if (!LSHB_OK(id >= a.id_base && (int64_t)(id - a.id_base) < a.n)) continue;   // (checked build only)
        const float* x = a.X + (int64_t)(id - a.id_base) * a.ldx;
        float s0 = 0.f, s1 = 0.f;   // L2: sum (x-q)^2 | cosine: x.q, |x|^2
        if (a.vec) {
            const float4* x4 = reinterpret_cast<const float4*>(x);
            const float4* q4 = reinterpret_cast<const float4*>(q);
            const int d4 = a.d >> 2;
            float t0 = 0.f, t1 = 0.f;   // second accumulators: two independent chains
            int c = lane;
            for (; c + 32 < d4; c += 64) {
                const float4 xv = __ldg(x4 + c), qv = __ldg(q4 + c);
                const float4 xw = __ldg(x4 + c + 32), qw = __ldg(q4 + c + 32);
                if (a.cosine) {
                    s0 = fmaf(xv.x, qv.x, fmaf(xv.y, qv.y, fmaf(xv.z, qv.z, fmaf(xv.w, qv.w, s0))));
                    s1 = fmaf(xv.x, xv.x, fmaf(xv.y, xv.y, fmaf(xv.z, xv.z, fmaf(xv.w, xv.w, s1))));
                    t0 = fmaf(xw.x, qw.x, fmaf(xw.y, qw.y, fmaf(xw.z, qw.z, fmaf(xw.w, qw.w, t0))));
                    t1 = fmaf(xw.x, xw.x, fmaf(xw.y, xw.y, fmaf(xw.z, xw.z, fmaf(xw.w, xw.w, t1))));
                } else {
                    const float d0 = xv.x - qv.x, d1 = xv.y - qv.y, d2 = xv.z - qv.z, d3 = xv.w - qv.w;
                    const float e0 = xw.x - qw.x, e1 = xw.y - qw.y, e2 = xw.z - qw.z, e3 = xw.w - qw.w;
                    s0 = fmaf(d0, d0, fmaf(d1, d1, fmaf(d2, d2, fmaf(d3, d3, s0))));
                    t0 = fmaf(e0, e0, fmaf(e1, e1, fmaf(e2, e2, fmaf(e3, e3, t0))));
                }
            }
            for (; c < d4; c += 32) {
                const float4 xv = __ldg(x4 + c), qv = __ldg(q4 + c);
                if (a.cosine) {
                    s0 = fmaf(xv.x, qv.x, fmaf(xv.y, qv.y, fmaf(xv.z, qv.z, fmaf(xv.w, qv.w, s0))));
                    s1 = fmaf(xv.x, xv.x, fmaf(xv.y, xv.y, fmaf(xv.z, xv.z, fmaf(xv.w, xv.w, s1))));
                } else {
                    const float d0 = xv.x - qv.x, d1 = xv.y - qv.y, d2 = xv.z - qv.z, d3 = xv.w - qv.w;
                    s0 = fmaf(d0, d0, fmaf(d1, d1, fmaf(d2, d2, fmaf(d3, d3, s0))));
                }
            }
            s0 += t0;
            s1 += t1;
        } else {
            for (int c = lane; c < a.d; c += 32) {
                const float xv = __ldg(x + c), qv = __ldg(q + c);
                if (a.cosine) {
                    s0 = fmaf(xv, qv, s0);
                    s1 = fmaf(xv, xv, s1);
                } else {
                    const float df = xv - qv;
                    s0 = fmaf(df, df, s0);
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, o);
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        }
        if (lane == 0) {
            float sc;
            if (a.cosine) {
                const float den = sqrtf(s1) * s_qn;
                sc = den > 0.f ? s0 / den : 0.f;
                sc = -sc;                  // descending similarity = ascending -similarity
                if (sc == 0.f) sc = 0.f;   // one zero
            } else {
                sc = s0;
            }
            key[j] = ((unsigned long long)ord_f32(sc) << 32) | id;
        }
    }
    for (int i = u + threadIdx.x; i < P; i += kQT) key[i] = ~0ull;
    __syncthreads();
    // 5. top-k
    bitonic_sort(key, P);
    for (int j = threadIdx.x; j < a.k; j += kQT) {
        int64_t id = -1;
        float sc = a.cosine ? -INFINITY : INFINITY;
        if (j < u) {
            const unsigned long long kv = key[j];
            id = (int64_t)(uint32_t)kv;
            sc = unord_f32((uint32_t)(kv >> 32));
            if (a.cosine) sc = -sc;
        }
        a.out_ids[qi * a.k + j] = id;
        a.out_score[qi * a.k + j] = sc;
    }
    if (threadIdx.x == 0 && a.out_ncand) a.out_ncand[qi] = (int32_t)s_u;
}

cudaError_t launch_knn(const IndexDev& idx, int64_t n, int L, uint32_t id_base, const int64_t* begin,
                       const int64_t* end, const float* X, int64_t ldx, int d, const float* Q, int64_t ldq,
                       int64_t nq, int k, int max_cand, int cosine, int64_t* out_ids, float* out_score,
                       int32_t* out_ncand, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    int P = 32;
    while (P < max_cand) P <<= 1;
    KnnArgs a;
    a.idx = idx;
    a.n = n;
    a.L = L;
    a.id_base = id_base;
    a.begin = begin;
    a.end = end;
    a.X = X;
    a.ldx = ldx;
    a.d = d;
    a.Q = Q;
    a.ldq = ldq;
    a.k = k;
    a.max_cand = max_cand;
    a.cosine = cosine;
    a.vec = (d % 4 == 0) && (ldx % 4 == 0) && (ldq % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0) &&
            ((reinterpret_cast<uintptr_t>(Q) & 15) == 0);
    a.out_ids = out_ids;
    a.out_score = out_score;
    a.out_ncand = out_ncand;
    const size_t smem = (size_t)P * 12 + (size_t)(L + 1) * 4;
    cudaError_t e = cudaFuncSetAttribute(knn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    knn_kernel<<<(unsigned)nq, kQT, smem, s>>>(a, P);
    return cudaGetLastError();
}

}  // namespace lshb
