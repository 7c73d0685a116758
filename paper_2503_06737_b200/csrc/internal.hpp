// internal.hpp — structures shared by the host core (api.cu) and the kernel
// launchers (sketch*.cu, group.cu, dense_tc.cu, knn.cu).  Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

// Device-side bounds checks of the checked build (build.py --variant checked,
// -DLSHB_CHECKS): LSHB_OK(cond) guards a write — a failed check prints the site and
// skips the write (tools/gpu_checked.sh greps for "LSHB_DCHECK").  In the product
// build it is `true` and vanishes.  (compute-sanitizer is closed on this GPU pool.)
#ifdef LSHB_CHECKS
#include <cstdio>
#define LSHB_OK(c) ((c) ? true : (printf("LSHB_DCHECK %s:%d\n", __FILE__, __LINE__), false))
#else
#define LSHB_OK(c) true
#endif

namespace lshb {

// ---------------------------------------------------------------------------
// Sparse one-nonzero-per-column projection (CS and HCS), DESIGN.md §K1.
// The host planner turns the per-coordinate (bin, sign) map of Def. CS
// / Def. HCS into, per coordinate chunk and per
// bin, the run of contributing coordinates: coordinates are staged in bin-sorted
// order (ascending coordinate inside a bin) with their sign already applied.
// ---------------------------------------------------------------------------
// Words per staged float4 column of the K1 tile (4 coordinates x 32 points + 4 pad):
// coordinate k of point r sits at word (k>>2)*kSketchColWords + (k&3)*32 + r.
constexpr int kSketchColWords = 132;

struct SketchPlanDev {
    int d, m, L, K;
    int Q;            // coordinates per chunk (64 * VPT)
    int vpt;          // float4 registers per thread (template selector: 1, 4, 16)
    int nchunks;
    int max_cnt;      // largest number of coordinates of one bin inside one chunk
    const uint16_t* pos;        // [d] staged-tile word offset of the coordinate at each bin-sorted index
    const uint32_t* bin_ptr;    // [nchunks][m+1] absolute index (chunk start + rank) where each bin starts
    const uint32_t* sign_bits;  // [ceil(d/32)] bit j set = sign(j) = -1 (applied while staging)
    const uint32_t* pairs;      // [2m] per bin: byte offsets (in the staged tile) of its first two coordinates,
                                //     lo 16 bits / hi 16 bits; missing ones point at the zero slot Q
    const uint32_t* fold_ptr;   // [L+1] table t's fold entries are fold[fold_ptr[t] .. fold_ptr[t+1])
    const uint32_t* fold;       // [nfold] (dst word << 16) | src word: the 3rd, 4th, ... coordinate of a bin is
                                //     added into its first coordinate's staged word before the pair gather
    int nfold;
};

// Chunked plan (sketch_chunked.cu): tables in groups, per group the coordinates
// whose bin is in the group, in chunks of <= 1024.
struct ChunkInfoDev {
    int32_t Qc;         // coordinates in this chunk
    int32_t t0, t1;     // tables of the chunk's group
    int32_t flags;      // bit 0: first chunk of the group, bit 1: last chunk of the group
    uint32_t coord_off; // offset of the chunk's first element in gcoord / pos / sgn
    uint32_t bp_off;    // offset of the chunk's (t1-t0)*K+1 bin starts in bp / cnt
    uint32_t pad0, pad1;
};
struct ChunkedPlanDev {
    int d, m, L, K;
    int nchunks;
    int gbins;        // largest group size in bins (partial-sum buffer)
    int max_cnt;      // largest coordinates-per-bin inside one chunk
    int vec_ok;       // every aligned group of 4 chunk elements is 4 contiguous, 16B-aligned inputs
    const ChunkInfoDev* chunks;
    const int32_t* gcoord;   // global input coordinate of every chunk element
    const uint16_t* pos;     // bin-sorted rank of every chunk element inside its chunk
    const uint32_t* sgn;     // sign bit of every chunk element
    const uint32_t* bp;      // bin start ranks (relative to the chunk)
    const uint8_t* cnt;      // coordinates per bin in the chunk (saturated at 255)
};

// HCS slab plan (sketch_hcs.cu): slab = d_1*d_2 contiguous inputs (one outer index
// J = (i_3..i_N)), adding into one block of M12 = m_1*m_2 bins; entries list the
// slabs block by block (empty blocks get one EMPTY entry).
#define HCS_BLOCK_MASK 0x1fffffffu
#define HCS_EMPTY (1u << 29)
#define HCS_NEG (1u << 30)
#define HCS_LAST (1u << 31)
struct HcsPlanDev {
    int m, K, S, M12;
    int nentries;
    const uint2* entries;    // .x = slab index J (input offset J*S), .y = block | flags
    const uint16_t* pos;     // [S] staged word offset of the coordinate at each bin-sorted position
    const uint32_t* sgn;     // [S/32] slab-internal sign bits (s_1 s_2 = -1)
    const uint16_t* bp;      // [M12+1] bin starts in the slab's bin-sorted order
    const uint8_t* wbins;    // [16][M12/16] bins of each warp (balanced by coordinate count)
    int nblocks;             // m / M12
    const int32_t* bfirst;   // [nblocks] index of each block's first entry
    int64_t d;               // input width (= product of the modes: the slab plan has no padding)
};

struct DiscretizeDev {
    int e2lsh;                // 1: E2LSH floor codes + fingerprint keys; 0: SRP bits
    float c_scale;            // sqrt(m)/w (CS/HCS), 1/w (dense)
    const float* c_off;       // [m] b_l / w  (E2LSH)
    int* flags;               // sticky device status (bit 0: int32 overflow, bit 1: NaN)
};

struct HashOut {
    uint64_t* keys;   // [L][n]
    int32_t* codes;   // [n][m]
    uint32_t* bits;   // [n][ceil(m/32)]
    float* proj;      // [n][m]
};

// Launchers (return cudaError_t of the launch).
cudaError_t launch_sketch(const SketchPlanDev& plan, const DiscretizeDev& disc, const float* X, int64_t n,
                          int64_t ld, HashOut out, int num_sms, cudaStream_t s);
cudaError_t launch_sketch_fast(const SketchPlanDev& plan, const DiscretizeDev& disc, const float* X, int64_t n,
                               int64_t ld, HashOut out, int num_sms, cudaStream_t s);
size_t sketch_smem_bytes(int Q, int m, int d, int L);
cudaError_t launch_sketch_chunked(const ChunkedPlanDev& plan, const DiscretizeDev& disc, const float* X, int64_t n,
                                  int64_t ld, HashOut out, int num_sms, cudaStream_t s);
size_t chunked_smem_bytes(int m, int gbins);
cudaError_t launch_sketch_hcs(const HcsPlanDev& plan, const DiscretizeDev& disc, const float* X, int64_t n,
                              int64_t ld, HashOut out, int num_sms, cudaStream_t s);
size_t hcs_smem_bytes(int S, int M12, int m, int nentries, int nst);
bool hcs_plan_supported(int S, int M12);

cudaError_t launch_dense_tc(const float* X, int64_t n, int64_t ld, int d, const uint16_t* R_pad, int m, int d_pad,
                            uint16_t* A_scratch, int64_t rows_per_batch, float* Y, cudaStream_t s,
                            uint64_t* keys = nullptr, int K = 0, const DiscretizeDev* dz = nullptr);
bool dense_tc_fused_keys_ok(int m, int K);
size_t dense_tc_rows_per_batch(int d_pad);
cudaError_t launch_keys_from_proj(const float* Y, int64_t n, int m, int L, int K, const DiscretizeDev& disc,
                                  HashOut out, cudaStream_t s);

// Grouping.
struct GroupScratch {
    uint64_t* keys_a;           // [L][n] keys after the L1 scatter
    uint32_t* ids_a;            // [L][n] ids after the L1 scatter
    uint32_t* hist;             // [L][nb1][tiles] per-tile L1 digit counts, then their tile scan
    uint32_t* tot;              // [L][nb1] bin totals
    uint32_t* binstart;         // [L][nb1+1]
    unsigned long long* state;  // [L][max(nb1, RLE chunks)] look-back words of the numbering
    uint32_t* perm;             // [L][2n] permutation scratch for bins larger than shared memory
    unsigned long long* vmask;  // [L][2] OR of keys, OR of complemented keys
    void* spec;                 // [2][L] L1 digit specs (group.cu)
    uint32_t* biglist;          // [L * nb1] L1 bins larger than the per-unit sort (wide keys)
    uint32_t* bigcount;         // [1]
    int num_sms;
};
struct IndexDev {
    uint32_t* ids;    // [L][n]
    uint64_t* ukeys;  // [L][n]  (capacity n per table)
    uint32_t* offs;   // [L][n+1]
    uint32_t* nb;     // [L]
};
size_t group_tiles(int64_t n);
int group_bins(int64_t n, int key_width);
size_t group_hist_words(int64_t n, int key_width);
size_t group_spec_bytes();
int group_rle_chunks(int64_t n);
size_t group_key_slots(int64_t n, int key_width);   // per-table L1 output slots
bool group_is_lsd(int key_width);
cudaError_t launch_group(const uint64_t* keys, int64_t n, int L, uint32_t id_base, int key_width,
                         GroupScratch& sc, IndexDev& out, int* flags, cudaStream_t s);
// interp: keys are 64-bit fingerprints (uniform): interpolation-guided probes first
cudaError_t launch_lookup(const uint64_t* qkeys, int64_t nq, int L, int64_t n, const IndexDev& idx,
                          int64_t* begin, int64_t* end, bool interp, cudaStream_t s);
cudaError_t launch_knn(const IndexDev& idx, int64_t n, int L, uint32_t id_base, const int64_t* begin,
                       const int64_t* end, const float* X, int64_t ldx, int d, const float* Q, int64_t ldq,
                       int64_t nq, int k, int max_cand, int cosine, int64_t* out_ids, float* out_score,
                       int32_t* out_ncand, cudaStream_t s);
cudaError_t launch_global_offsets(const uint32_t* all, int G, int rank, int L, int B, int64_t* off, cudaStream_t s);
cudaError_t launch_query_runs(const int64_t* all, int G, int rank, int64_t M, int64_t* gbegin, int64_t* gtotal,
                              cudaStream_t s);
cudaError_t launch_counts(const IndexDev& idx, int64_t n, int L, int width, int B, uint32_t* counts,
                          cudaStream_t s);

// Instrumentation (api.cu): every launch goes through these.
void timing_begin(const char* name, cudaStream_t s);
void timing_end(const char* name, cudaStream_t s);
void count_launch();

}  // namespace lshb
