/*
 * lsh.h — C ABI of the B200 (sm_100a) hot path of arXiv 2503.06737,
 * "Faster and Space Efficient Indexing for Locality Sensitive Hashing".
 *
 * The library hashes batches of d-dimensional fp32 points with the paper's
 * sketch-based hashers and builds the (m, L) hash-table index from the codes:
 *
 *   CS-E2LSH   g(p)_l  = floor((sqrt(m) CS(p)_l + b_l) / w)        PAPER.md:314  Def. CS-E2LSH
 *   HCS-E2LSH  g'(p)_l = floor((sqrt(m) vec(HCS(p))_l + b_l) / w)  PAPER.md:624  eq:eq_hca_eucl_lsh
 *   CS-SRP     xi(u)_l  = [CS(u)_l > 0]                            PAPER.md:918  Def. CS-SRP
 *   HCS-SRP    xi'(u)_l = [vec(HCS(u))_l > 0]                      PAPER.md:1441 Def. HCS-SRP
 *   E2LSH      h(p)_l  = floor((<r_l,p> + b_l) / w)               PAPER.md:169  eq:datar_lsh (dense baseline)
 *   SRP        zeta(u)_l = [<r_l,u> > 0]                           PAPER.md:187  Def. SRP      (dense baseline)
 *
 * with CS(p)_l = sum_{h(i)=l} s(i) p_i (eq:eq_cs) and
 * HCS(p)_{l_1..l_N} = sum_{h_k(i_k)=l_k} prod_k s_k(i_k) p_j (eq:eqhcs).
 * The index stores every point p in bucket hbar_t(p) of each table t (§3.1).
 *
 * Readings of the paper this interface fixes:
 *   - m is the total code size and m = L*K; table t uses code coordinates
 *     [t*K, (t+1)*K) of ONE sketch per point (B1).  sqrt(m) uses that total m (B2).
 *   - one offset b_l ~ U[0, w) per code coordinate (B3, B4).
 *   - HCS reshapes with 0-based column-major (i_1 fastest) index maps, zero padding
 *     when prod d_k > d (B6, B7).
 *   - A table's bucket key: SRP = the K bits packed little-endian (bit k of the key =
 *     code coordinate t*K+k), exact; E2LSH = 64-bit fingerprint of the K int32 codes
 *     u_k (two's-complement words): lanes a = sum u_k A^(K-1-k), b = sum u_k B^(K-1-k)
 *     mod 2^32 (A = 0x9E3779B1, B = 0x85EBCA77), key = SplitMix64-finaliser(a:b) (B10).
 *   - Inside a table, buckets are ordered by ascending unsigned key and ids ascend
 *     inside a bucket (B11).
 *   - Random parameters derive from `seed` exactly as DESIGN.md R1-R4 state
 *     (SplitMix64 streams keyed by FNV-1a of a label, Mersenne-61 2-wise families,
 *     fp32 offsets, Box-Muller Gaussians rounded to bf16).
 *
 * Conventions for every function:
 *   - Returns lsh_status (0 = LSH_OK).  No function throws or aborts.
 *   - Pointers named X, Q, keys, codes, bits, proj, begin, end, counts are DEVICE
 *     pointers (CUDA global memory of params.device) owned by the caller; the
 *     library never frees caller memory.  `stream` is a cudaStream_t (NULL = legacy
 *     default stream) passed as void* so this header needs no CUDA include.
 *   - Device calls are stream-ordered and asynchronous (no host synchronisation)
 *     unless stated otherwise.  Handles and built indexes are immutable and may be
 *     used concurrently from several streams: every index consumer (queries, counts)
 *     first makes its stream wait for the index's build, and lsh_index_destroy orders
 *     the release of the index memory after the last use on every such stream.
 *   - X is row-major fp32 [n][ld], ld >= d (elements), rows contiguous.
 *   - Errors: LSH_EINVAL invalid parameters (w <= 0, m != L*K, prod mode_m != m,
 *     prod mode_d < d, K > 64 for SRP, m > 2^20, d > 2^27, N outside 1..8);
 *     LSH_EDIM n < 0, ld < d, nq < 0 or a size mismatch; LSH_ENOMEM allocation
 *     failure; LSH_ECUDA a CUDA runtime error (lsh_last_cuda_error() has the text);
 *     LSH_EOVERFLOW an E2LSH code outside int32 was produced (reported by lsh_check;
 *     the code is clamped, never silently wrapped); LSH_ESTATE misuse (NULL handle);
 *     LSH_EUNSUPPORTED a shape this build has no kernel for.
 */
#ifndef PAPER_2503_06737_LSH_H
#define PAPER_2503_06737_LSH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LSH_E2LSH = 0,      /* dense Gaussian projection, O(md)   (PAPER.md:166 Def. E2LSH) */
    LSH_SRP = 1,        /* dense Gaussian projection, O(md)   (PAPER.md:185 Def. SRP)   */
    LSH_CS_E2LSH = 2,   /* count sketch, O(d)            */
    LSH_CS_SRP = 3,     /* count sketch, O(d)            */
    LSH_HCS_E2LSH = 4,  /* higher-order count sketch, O(d)            */
    LSH_HCS_SRP = 5     /* higher-order count sketch, O(d)           */
} lsh_scheme;

typedef enum {
    LSH_OK = 0,
    LSH_EINVAL = 1,
    LSH_EDIM = 2,
    LSH_ENOMEM = 3,
    LSH_ECUDA = 4,
    LSH_EOVERFLOW = 5,
    LSH_ESTATE = 6,
    LSH_EUNSUPPORTED = 7
} lsh_status;

#define LSH_MAX_MODES 8

/* Problem statement (PAPER.md:23 d, m; :166-171 w, b, r; :202-216 h, s, N, d_k, m_k;
 * :155 number of tables).  Plain-old-data; field order is part of the ABI. */
typedef struct {
    int32_t scheme;                 /* lsh_scheme */
    int32_t N;                      /* HCS tensor order 1..8; must be 1 for CS and dense */
    int64_t d;                      /* input dimension, >= 1 */
    int32_t mode_d[LSH_MAX_MODES];  /* HCS: d_1..d_N with prod >= d (zero padding); CS/dense: mode_d[0] = d */
    int32_t mode_m[LSH_MAX_MODES];  /* HCS: m_1..m_N with prod == m;                CS/dense: mode_m[0] = m */
    int32_t m;                      /* total code size, == L*K */
    int32_t L;                      /* number of hash tables */
    int32_t K;                      /* code coordinates per table (SRP: K <= 64) */
    float w;                        /* bucket width, > 0 (E2LSH family; ignored by SRP) */
    uint64_t seed;                  /* master seed of every random draw */
    int32_t device;                 /* CUDA device ordinal */
    int32_t flags;                  /* LSH_FLAG_* bits; other bits must be 0 */
} lsh_params;

/* NEXT-2, reading C3: "L independent hash tables of m-sized
 * hash codes" taken literally -- table t has its own count sketch of
 * size K: h_t : [d] -> [K], s_t : [d] -> {+1,-1}, offsets b_t[K], drawn from the
 * streams "table{t}/mode0/bucket", "table{t}/mode0/sign", "table{t}/offsets";
 * code coordinate tK + k is floor((sqrt(K) CS_t(x)_k + b_tk) / w) (E2LSH) or
 * [CS_t(x)_k > 0] (SRP).  CS schemes only (others: LSH_EUNSUPPORTED).  O(L d) adds
 * per point; this build runs it as one tensor-core GEMM with the K-sparse +-1
 * matrix [m][d] (exact in bf16) and the dense path's 3-term bf16 split of x. */
#define LSH_FLAG_PER_TABLE 1

typedef struct lsh_handle lsh_handle;  /* hasher: parameters resident on the device */
typedef struct lsh_index lsh_index;    /* built (m, L) index, device-resident CSR per table */

/* ---- lifetime ----------------------------------------------------------- */

/* Validate `p`, draw every random parameter on the host (R1-R4), build the
 * device execution plan and upload it.  Synchronous (the only call that is).
 * On success *out owns ~O(d) (CS), O(sum d_k + d) (HCS) or O(md) (dense) device bytes. */
lsh_status lsh_create(const lsh_params* p, lsh_handle** out);
void lsh_destroy(lsh_handle* h);

/* ---- hashing (§8(a) rows a-2..a-4) -------------------------------------- */

/* Hash rows X[0..n) on `stream`.  Any output may be NULL (skipped):
 *   keys  uint64 [L][n]            table keys (row t = table t), see B10 above
 *   codes int32  [n][m]            E2LSH schemes only: the integer codes
 *   bits  uint32 [n][ceil(m/32)]   SRP schemes only: bit l of point i at word l/32, bit l%32
 *   proj  float  [n][m]            debug: the pre-discretisation projection
 *                                  (CS / vec(HCS) / <r_l, x>) in fp32
 * Requires n >= 0, ld >= d.  Asynchronous. */
lsh_status lsh_hash(const lsh_handle* h, const float* X, int64_t n, int64_t ld,
                    uint64_t* keys, int32_t* codes, uint32_t* bits, float* proj, void* stream);

/* ---- index (§8(a) rows a-5, a-7) ---------------------------------------- */

/* Hash X and group the n points into the buckets of every table; point i gets the
 * global id (id_base + i) (uint32; id_base + n <= 2^32 - 1: 0xffffffff is reserved).  n == 0 gives an empty
 * index.  Asynchronous: *out is valid immediately, its contents after `stream`
 * reaches this point. */
lsh_status lsh_build_index(const lsh_handle* h, const float* X, int64_t n, int64_t ld,
                           int64_t id_base, lsh_index** out, void* stream);

/* Group given keys [L][n] (device) as lsh_build_index does after hashing
 * (grouping-parity entry: feed the oracle's keys, compare the tables). */
lsh_status lsh_group_keys(const lsh_handle* h, const uint64_t* keys, int64_t n,
                          int64_t id_base, lsh_index** out, void* stream);

/* Device pointers of table t (valid until lsh_index_destroy) and its bucket count:
 *   ids   uint32 [n]      ids sorted by (key, id)
 *   ukeys uint64 [nb]     distinct keys ascending
 *   offs  uint32 [nb+1]   bucket b = ids[offs[b] .. offs[b+1])
 * Synchronises with the index's build (host needs nb). */
lsh_status lsh_index_view(const lsh_index* idx, int32_t t, const uint32_t** ids,
                          const uint64_t** ukeys, const uint32_t** offs, int64_t* nb);
int64_t lsh_index_size(const lsh_index* idx);   /* n of the build, -1 on NULL */
void lsh_index_destroy(lsh_index* idx);

/* Hash queries Q [nq][ld] and look their key up in every table:
 * begin/end int64 [nq][L] (device) = the bucket's [offs[b], offs[b+1]) in table t,
 * or an empty range begin == end == offs[insertion point] when the key is absent. */
lsh_status lsh_query_buckets(const lsh_handle* h, const lsh_index* idx, const float* Q,
                             int64_t nq, int64_t ld, int64_t* begin, int64_t* end, void* stream);

/* Query completion ("collect the index of all the
 * elements", §6 PAPER.md:2000-2003 top-k retrieval).  For each query: its L bucket
 * ranges (as lsh_query_buckets), the bucket entries in table order capped at
 * max_cand entries, distinct ids, exact re-rank against the indexed points and the
 * top k.  Similarity: squared Euclidean distance, ascending, for the E2LSH family;
 * cosine similarity, descending, for the SRP family (0 when a norm is 0); ties by
 * ascending id (readings C1, C2 in DESIGN.md).
 *   X       float [n][ldx] (device): the rows the index was built from; id i is row
 *           i - id_base of X (the caller keeps X alive; the library reads it).
 *   Q       float [nq][ldq] (device) queries, ldq >= d.
 *   out_ids int64 [nq][k] (device): ids, -1 where fewer than k candidates.
 *   out_score float [nq][k] (device): the scores (+inf / -inf in missing slots).
 *   out_ncand int32 [nq] (device, nullable): distinct candidates examined.
 * 1 <= k <= max_cand <= 8192 (LSH_EINVAL otherwise); ldx, ldq >= d (LSH_EDIM).
 * Asynchronous on `stream`; temporaries are stream-ordered allocations. */
lsh_status lsh_query_knn(const lsh_handle* h, const lsh_index* idx, const float* X, int64_t ldx, const float* Q,
                         int64_t nq, int64_t ldq, int32_t k, int32_t max_cand, int64_t* out_ids, float* out_score,
                         int32_t* out_ncand, void* stream);

/* Coarse per-table histogram for the multi-GPU exchange (§8(e)): counts uint32
 * [L][2^B] (device, overwritten), bin = top B bits of the key's significant width
 * (64 for E2LSH fingerprints, K for SRP; the key itself when that width <= B).
 * 1 <= B <= 20. */
lsh_status lsh_index_counts(const lsh_index* idx, int32_t B, uint32_t* counts, void* stream);

/* Multi-GPU exchange step (§8(e)): given the all-gathered coarse counts of every rank,
 * all_counts uint32 [G][L][2^B] (device), write offsets int64 [L][2^B] (device): the
 * global position where rank `rank`'s run of (table t, coarse bin b) starts in the
 * global bin-major / rank-minor order,
 *   offsets[t][b] = sum_{b'<b} sum_r all_counts[r][t][b'] + sum_{r'<rank} all_counts[r'][t][b].
 * 0 <= rank < G, 1 <= B <= 20.  Asynchronous. */
lsh_status lsh_global_offsets(const uint32_t* all_counts, int32_t G, int32_t rank, int32_t L, int32_t B,
                              int64_t* offsets, void* stream);

/* Cross-shard query (§8(e); "collect the index of all the elements"
 * hashed to hbar_t(q), over every shard).  Each rank looks its queries up in its own
 * tables (lsh_query_buckets: local begin/end [nq][L]); the ranges of all ranks are
 * all-gathered as all_ranges int64 [G][2][M] (device; rank r's begin[M] then end[M],
 * M = nq*L).  Because the global bucket of (q, t) is the rank-order concatenation of
 * the ranks' runs (global ids ascend across ranks), rank `rank`'s local entries
 * ids[begin[j], end[j]) sit at positions
 *   gbegin[j] = sum_{r < rank} (end_r[j] - begin_r[j])   (int64 [M], device, written)
 * of that global bucket, whose size is gtotal[j] = sum_r (end_r[j] - begin_r[j])
 * (int64 [M], device, nullable).  0 <= rank < G, M >= 0 (LSH_EDIM otherwise).
 * Asynchronous on `stream`. */
lsh_status lsh_query_global_runs(const int64_t* all_ranges, int32_t G, int32_t rank, int64_t M, int64_t* gbegin,
                                 int64_t* gtotal, void* stream);

/* ---- parameters, errors, instrumentation -------------------------------- */

typedef enum {
    LSH_EXPORT_BUCKET = 0,    /* int32 [d_k]  h_k of mode `mode` (CS: mode 0 = h)           */
    LSH_EXPORT_SIGN = 1,      /* int32 [d_k]  s_k of mode `mode`, values +1 / -1            */
    LSH_EXPORT_OFFSETS = 2,   /* float [m]    b_l                                           */
    LSH_EXPORT_GAUSSIAN = 3,  /* uint16 [m*d] bf16 bit patterns of R, row-major (dense)    */
    LSH_EXPORT_COEFFS = 4,    /* uint64 [4]   (a, b) of mode `mode`'s bucket then sign family */
    LSH_EXPORT_COORD = 5      /* int32 [2*d]  per input coordinate j: bin, then sign        */
} lsh_export_what;

/* Host-only parameter draw (no CUDA call): writes the requested table into host_buf.
 * If host_buf is NULL or *bytes is too small, sets *bytes to the size needed and
 * returns LSH_EDIM (nothing written). */
lsh_status lsh_export_host(const lsh_params* p, int32_t what, int32_t mode, void* host_buf, size_t* bytes);

/* Same tables read back from the handle's DEVICE copies (synchronous D2H). */
lsh_status lsh_get_params(const lsh_handle* h, int32_t what, int32_t mode, void* host_buf, size_t* bytes);

/* Synchronise the handle's device and return the sticky device status
 * (LSH_EOVERFLOW if any E2LSH code left int32 since the last lsh_check). */
lsh_status lsh_check(const lsh_handle* h);

/* Grouping path of the handle's wide-key builds (E2LSH fingerprints, SRP with K > 22),
 * DESIGN.md §7 K3; diagnostics only (both paths give the same canonical index, B11).
 * Synchronises the handle's device.  *path = 0: the fixed-capacity L1 scatter (keys
 * read once, no histogram pass); > 0: a recent build overflowed a bin (duplicate-heavy
 * codes) and builds currently take the histogram path (the value counts down over the
 * next builds).  Narrow keys always take the LSD path (*path = 0).  LSH_ESTATE if
 * h or path is NULL. */
lsh_status lsh_group_path(const lsh_handle* h, int32_t* path);

const char* lsh_strerror(lsh_status s);
const char* lsh_last_cuda_error(void);

/* Total number of CUDA kernels this library has launched (process-wide). */
uint64_t lsh_launch_count(void);

/* Per-kernel device time: when enabled, every internal launch on a handle is
 * bracketed by CUDA events on its stream and accumulated by kernel name. */
void lsh_timing_enable(int32_t on);
/* Names: "sketch", "sketch_query", "dense_gemm", "dense_gemm_query", "keys_from_proj",
 * "group_hist", "group_scan", "group_scatter", "group_sort", "lookup", "knn", "counts",
 * "global_offsets", "query_runs".  Synchronises the device.
 * Returns accumulated milliseconds and launch count since the last reset. */
lsh_status lsh_timing_get(const char* name, double* ms, int64_t* launches);
void lsh_timing_reset(void);

#ifdef __cplusplus
}
#endif
#endif /* PAPER_2503_06737_LSH_H */
