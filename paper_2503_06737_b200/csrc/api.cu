// api.cu — host core of the C ABI declared in include/lsh.h.
//
// Validates the problem statement, draws the random parameters on the host
// (params.hpp, R1-R4), plans the device execution (per-chunk bin lists
// for the sketch kernel), owns device buffers of handles and indexes, and
// launches the kernels of sketch*.cu / dense_tc.cu / group.cu / knn.cu on the caller's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/lsh.h"
#include "internal.hpp"
#include "params.hpp"

using namespace lshb;

// ---------------------------------------------------------------------------
// errors, launch counting, timing
// ---------------------------------------------------------------------------
static std::mutex g_err_mu;
static std::string g_last_cuda_error = "";
static std::atomic<uint64_t> g_launches{0};

static lsh_status cuda_fail(cudaError_t e, const char* where) {
    std::lock_guard<std::mutex> g(g_err_mu);
    g_last_cuda_error = std::string(where) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? LSH_ENOMEM : LSH_ECUDA;
}
#define CK(call)                                              \
    do {                                                      \
        cudaError_t e_ = (call);                              \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);   \
    } while (0)

namespace lshb {
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

struct TimingSlot {
    double ms = 0;
    int64_t launches = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
    cudaEvent_t open = nullptr;
};
static std::mutex g_time_mu;
static std::atomic<int> g_timing_on{0};
static std::map<std::string, TimingSlot> g_slots;
static std::vector<cudaEvent_t> g_event_pool;

static cudaEvent_t get_event() {
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
void timing_begin(const char* name, cudaStream_t s) {
    if (!g_timing_on.load()) return;
    std::lock_guard<std::mutex> g(g_time_mu);
    TimingSlot& sl = g_slots[name];
    sl.open = get_event();
    cudaEventRecord(sl.open, s);
}
void timing_end(const char* name, cudaStream_t s) {
    if (!g_timing_on.load()) return;
    std::lock_guard<std::mutex> g(g_time_mu);
    TimingSlot& sl = g_slots[name];
    if (!sl.open) return;
    cudaEvent_t e = get_event();
    cudaEventRecord(e, s);
    sl.pending.emplace_back(sl.open, e);
    sl.open = nullptr;
    sl.launches++;
}
}  // namespace lshb

extern "C" uint64_t lsh_launch_count(void) { return g_launches.load(); }
extern "C" void lsh_timing_enable(int32_t on) { g_timing_on.store(on ? 1 : 0); }
extern "C" void lsh_timing_reset(void) {
    std::lock_guard<std::mutex> g(g_time_mu);
    for (auto& kv : g_slots) {
        for (auto& pr : kv.second.pending) {
            g_event_pool.push_back(pr.first);
            g_event_pool.push_back(pr.second);
        }
        kv.second = TimingSlot();
    }
}
extern "C" lsh_status lsh_timing_get(const char* name, double* ms, int64_t* launches) {
    CK(cudaDeviceSynchronize());
    std::lock_guard<std::mutex> g(g_time_mu);
    auto it = g_slots.find(name);
    if (it == g_slots.end()) {
        if (ms) *ms = 0;
        if (launches) *launches = 0;
        return LSH_OK;
    }
    TimingSlot& sl = it->second;
    for (auto& pr : sl.pending) {
        float t = 0;
        cudaEventElapsedTime(&t, pr.first, pr.second);
        sl.ms += t;
        g_event_pool.push_back(pr.first);
        g_event_pool.push_back(pr.second);
    }
    sl.pending.clear();
    if (ms) *ms = sl.ms;
    if (launches) *launches = sl.launches;
    return LSH_OK;
}

extern "C" const char* lsh_last_cuda_error(void) {
    static thread_local std::string copy;
    std::lock_guard<std::mutex> g(g_err_mu);
    copy = g_last_cuda_error;
    return copy.c_str();
}

extern "C" const char* lsh_strerror(lsh_status s) {
    switch (s) {
        case LSH_OK: return "ok";
        case LSH_EINVAL: return "invalid parameters";
        case LSH_EDIM: return "invalid dimension or size";
        case LSH_ENOMEM: return "out of device memory";
        case LSH_ECUDA: return "CUDA error";
        case LSH_EOVERFLOW: return "E2LSH code outside int32";
        case LSH_ESTATE: return "invalid handle or state";
        case LSH_EUNSUPPORTED: return "unsupported shape for this build";
    }
    return "unknown status";
}

// ---------------------------------------------------------------------------
// parameter validation and the host-side draw
// ---------------------------------------------------------------------------
static bool is_dense(int s) { return s == LSH_E2LSH || s == LSH_SRP; }
static bool is_hcs(int s) { return s == LSH_HCS_E2LSH || s == LSH_HCS_SRP; }
static bool is_e2lsh(int s) { return s == LSH_E2LSH || s == LSH_CS_E2LSH || s == LSH_HCS_E2LSH; }

static lsh_status validate(const lsh_params* p) {
    if (!p) return LSH_ESTATE;
    if (p->scheme < 0 || p->scheme > 5) return LSH_EINVAL;
    if (p->d < 1 || p->d > (1ll << 27)) return LSH_EINVAL;
    if (p->m < 1 || p->m > (1 << 20) || p->L < 1 || p->K < 1) return LSH_EINVAL;
    if ((int64_t)p->L * p->K != p->m) return LSH_EINVAL;
    if (!(p->w > 0.0f) || !std::isfinite(p->w)) return LSH_EINVAL;
    if (!is_e2lsh(p->scheme) && p->K > 64) return LSH_EINVAL;
    if (p->flags & ~LSH_FLAG_PER_TABLE) return LSH_EINVAL;
    // dense R / per-table sign matrix: m*d bf16 on the host and the device (<= 32 GiB)
    if ((is_dense(p->scheme) || (p->flags & LSH_FLAG_PER_TABLE)) && (int64_t)p->m * p->d > (1ll << 34))
        return LSH_EINVAL;
    if ((p->flags & LSH_FLAG_PER_TABLE) && !(p->scheme == LSH_CS_E2LSH || p->scheme == LSH_CS_SRP))
        return LSH_EUNSUPPORTED;
    if (is_hcs(p->scheme)) {
        if (p->N < 1 || p->N > LSH_MAX_MODES) return LSH_EINVAL;
        int64_t pd = 1, pm = 1;
        for (int k = 0; k < p->N; ++k) {
            if (p->mode_d[k] < 1 || p->mode_m[k] < 1) return LSH_EINVAL;
            pd *= p->mode_d[k];
            pm *= p->mode_m[k];
            if (pd > (1ll << 40)) return LSH_EINVAL;
        }
        if (pm != p->m || pd < p->d) return LSH_EINVAL;
    } else {
        if (p->N != 1) return LSH_EINVAL;
    }
    return LSH_OK;
}

struct HostTables {
    int N = 1;
    std::vector<int64_t> md, mm;             // mode sizes
    std::vector<std::vector<int32_t>> h, s;  // per mode
    std::vector<TwoWise> fb, fs;             // per mode families
    std::vector<float> b;
    std::vector<uint16_t> R;                 // dense only, bf16 bits [m][d]
};

static bool is_per_table(const lsh_params* p) { return (p->flags & LSH_FLAG_PER_TABLE) != 0; }
// dense projection matrix in the handle: the Gaussian R, or the per-table sign matrix
static bool uses_R(const lsh_params* p) { return is_dense(p->scheme) || is_per_table(p); }

static void draw(const lsh_params* p, HostTables& t, bool with_gaussian) {
    if (is_per_table(p)) {
        // reading C3: table t draws (h_t, s_t, b_t) from its own "table{t}/" streams; the
        // matrix row tK + h_t(i), column i holds s_t(i) (bf16 +-1, exact)
        t.N = p->L;
        t.b.clear();
        t.R.assign((size_t)p->m * p->d, 0);
        for (int tt = 0; tt < p->L; ++tt) {
            const std::string pre = "table" + std::to_string(tt) + "/";
            TwoWise fb = bucket_family(p->seed, 0, (uint64_t)p->K, pre);
            TwoWise fs = sign_family(p->seed, 0, pre);
            std::vector<float> bt;
            offsets(p->seed, p->K, p->w, bt, pre);
            t.b.insert(t.b.end(), bt.begin(), bt.end());
            std::vector<int32_t> hv(p->d), sv(p->d);
            for (int64_t i = 0; i < p->d; ++i) {
                hv[i] = (int32_t)fb.eval((uint64_t)i);
                sv[i] = fs.eval((uint64_t)i) == 0 ? 1 : -1;
                t.R[(size_t)(tt * p->K + hv[i]) * p->d + i] = sv[i] > 0 ? 0x3F80 : 0xBF80;
            }
            t.md.push_back(p->d);
            t.mm.push_back(p->K);
            t.fb.push_back(fb);
            t.fs.push_back(fs);
            t.h.push_back(std::move(hv));
            t.s.push_back(std::move(sv));
        }
        return;
    }
    offsets(p->seed, p->m, p->w, t.b);
    if (is_dense(p->scheme)) {
        t.N = 1;
        if (with_gaussian) {
            const int64_t total = (int64_t)p->m * p->d;
            t.R.assign(total, 0);
            const int64_t pairs = (total + 1) / 2;
            unsigned nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
            if (pairs < 65536) nth = 1;
            std::vector<std::thread> th;
            for (unsigned k = 0; k < nth; ++k) {
                const int64_t lo = pairs * k / nth, hi = pairs * (k + 1) / nth;
                th.emplace_back([&, lo, hi]() { gaussian_range(p->seed, total, lo, hi, t.R.data()); });
            }
            for (auto& x : th) x.join();
        }
        return;
    }
    t.N = is_hcs(p->scheme) ? p->N : 1;
    for (int k = 0; k < t.N; ++k) {
        const int64_t dk = is_hcs(p->scheme) ? p->mode_d[k] : p->d;
        const int64_t mk = is_hcs(p->scheme) ? p->mode_m[k] : p->m;
        t.md.push_back(dk);
        t.mm.push_back(mk);
        TwoWise fb = bucket_family(p->seed, k, (uint64_t)mk);
        TwoWise fs = sign_family(p->seed, k);
        t.fb.push_back(fb);
        t.fs.push_back(fs);
        std::vector<int32_t> hv(dk), sv(dk);
        for (int64_t i = 0; i < dk; ++i) {
            hv[i] = (int32_t)fb.eval((uint64_t)i);
            sv[i] = fs.eval((uint64_t)i) == 0 ? 1 : -1;
        }
        t.h.push_back(std::move(hv));
        t.s.push_back(std::move(sv));
    }
}

// Per input coordinate j < d: the bin it adds to and its sign (Def. CS: h(j), s(j);
// Def. HCS: l = sum_k h_k(i_k) prod_{t<k} m_t, sign = prod_k s_k(i_k) with
// (i_1..i_N) the column-major unflatten of j).
static void coordinate_map(const lsh_params* p, const HostTables& t, std::vector<int32_t>& bin,
                           std::vector<int8_t>& sgn) {
    bin.resize(p->d);
    sgn.resize(p->d);
    for (int64_t j = 0; j < p->d; ++j) {
        int64_t rem = j, l = 0, stride = 1;
        int sg = 1;
        for (int k = 0; k < t.N; ++k) {
            const int64_t ik = rem % t.md[k];
            rem /= t.md[k];
            l += (int64_t)t.h[k][ik] * stride;
            stride *= t.mm[k];
            sg *= t.s[k][ik];
        }
        bin[j] = (int32_t)l;
        sgn[j] = (int8_t)sg;
    }
}

// ---------------------------------------------------------------------------
// handle
// ---------------------------------------------------------------------------
struct lsh_handle {
    lsh_params p{};
    HostTables host;
    int device = 0, num_sms = 148;
    int key_width = 64;
    SketchPlanDev plan{};
    DiscretizeDev disc{};
    bool chunked = false;
    ChunkedPlanDev cplan{};
    void* d_cplan_mem = nullptr;
    uint16_t* d_entries = nullptr;
    uint32_t* d_binptr = nullptr;
    uint32_t* d_signs = nullptr;
    uint32_t* d_pairs = nullptr;
    uint32_t* d_fold = nullptr;     // [L+1] fold_ptr, then [nfold] fold entries
    float* d_coff = nullptr;
    uint16_t* d_R = nullptr;
    uint16_t* d_Rpad = nullptr;  // bf16 [m][d_pad], d_pad = roundup(d, 64): tensor-core B operand
    int d_pad = 0;
    int* d_flags = nullptr;
    std::vector<int32_t*> d_h, d_s;
    float* d_b = nullptr;
    bool sketch_ok = true;
    bool hcs = false;          // HCS slab plan available (sketch_hcs.cu)
    HcsPlanDev hplan{};
    void* d_hplan_mem = nullptr;
};

struct lsh_index {
    const lsh_handle* h = nullptr;
    int64_t n = 0;
    int64_t id_base = 0;
    int L = 0;
    IndexDev dev{};
    void* mem = nullptr;
    cudaEvent_t done = nullptr;
    cudaStream_t stream = nullptr;  // build stream: memory is freed stream-ordered on it
    // Consumers on other streams (queries, counts): each waits on `done` before reading,
    // and records a last-use event here, so destroy can order the stream-ordered free
    // after every reader without a host synchronisation.
    mutable std::mutex use_mu;
    mutable std::vector<std::pair<cudaStream_t, cudaEvent_t>> uses;
};

// Start of an index consumer on stream s: the build must be complete.
static cudaError_t index_acquire(const lsh_index* I, cudaStream_t s) { return cudaStreamWaitEvent(s, I->done, 0); }
// End of an index consumer on stream s: remember the stream's last use.
static void index_release(const lsh_index* I, cudaStream_t s) {
    if (s == I->stream) return;   // the free is stream-ordered on the build stream already
    std::lock_guard<std::mutex> g(I->use_mu);
    for (auto& u : I->uses)
        if (u.first == s) {
            cudaEventRecord(u.second, s);
            return;
        }
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return;
    cudaEventRecord(e, s);
    I->uses.emplace_back(s, e);
}

// Chunked plan (large d and/or m): tables in groups whose partial sums fit in
// shared memory; per group, the coordinates whose bin lies in the group (ascending),
// cut into chunks of <= 1024; per chunk, bin-sorted ranks.  See sketch_chunked.cu.
static lsh_status build_chunked_plan(lsh_handle* H, const std::vector<int32_t>& bin, const std::vector<int8_t>& sgn) {
    const lsh_params* p = &H->p;
    const int d = (int)p->d, m = p->m, K = p->K, L = p->L;
    const int Q = 1024;
    const size_t budget = 232448;
    int tables_per_group = 0;
    for (int g = L; g >= 1; --g) {
        if (chunked_smem_bytes(m, g * K) <= budget) {
            tables_per_group = g;
            break;
        }
    }
    if (tables_per_group == 0) {
        H->sketch_ok = false;
        return LSH_OK;
    }
    // coordinates of each group in ascending order
    const int ngroups = (L + tables_per_group - 1) / tables_per_group;
    std::vector<std::vector<int32_t>> gcoords(ngroups);
    for (int j = 0; j < d; ++j) gcoords[(bin[j] / K) / tables_per_group].push_back(j);
    std::vector<ChunkInfoDev> chunks;
    std::vector<int32_t> gcoord;
    std::vector<uint16_t> pos;
    std::vector<uint32_t> sgnb;
    std::vector<uint32_t> bp;
    std::vector<uint8_t> cnt;
    int max_cnt = 0, gbins = 0;
    bool vec_ok = true;
    for (int g = 0; g < ngroups; ++g) {
        const int t0 = g * tables_per_group, t1 = std::min(L, t0 + tables_per_group);
        const int nb = (t1 - t0) * K, b0 = t0 * K;
        gbins = std::max(gbins, nb);
        const std::vector<int32_t>& cl = gcoords[g];
        const int total = (int)cl.size();
        const int nck = std::max(1, (total + Q - 1) / Q);
        for (int c = 0; c < nck; ++c) {
            const int k0 = c * Q, k1 = std::min(total, k0 + Q);
            ChunkInfoDev ci{};
            ci.Qc = k1 - k0;
            ci.t0 = t0;
            ci.t1 = t1;
            ci.flags = (c == 0 ? 1 : 0) | (c == nck - 1 ? 2 : 0);
            ci.coord_off = (uint32_t)gcoord.size();
            ci.bp_off = (uint32_t)bp.size();
            std::vector<uint32_t> cn(nb + 1, 0);
            for (int k = k0; k < k1; ++k) cn[bin[cl[k]] - b0 + 1]++;
            for (int b = 0; b < nb; ++b) {
                max_cnt = std::max(max_cnt, (int)cn[b + 1]);
                cnt.push_back((uint8_t)std::min<uint32_t>(cn[b + 1], 255));
            }
            cnt.push_back(0);
            for (int b = 0; b < nb; ++b) cn[b + 1] += cn[b];
            for (int b = 0; b <= nb; ++b) bp.push_back(cn[b]);
            std::vector<uint32_t> cur(cn.begin(), cn.end() - 1);
            for (int k = k0; k < k1; ++k) {
                const int j = cl[k];
                const size_t idx = gcoord.size();
                gcoord.push_back(j);
                pos.push_back((uint16_t)cur[bin[j] - b0]++);
                if (sgnb.size() * 32 <= idx) sgnb.push_back(0);
                if (sgn[j] < 0) sgnb[idx >> 5] |= 1u << (idx & 31);
            }
            // 128-bit staging needs every aligned group of 4 elements to be 4 contiguous
            // inputs starting at a multiple of 4
            if (ci.Qc % 4) vec_ok = false;
            for (int k = 0; k + 3 < ci.Qc && vec_ok; k += 4) {
                const int j = cl[k0 + k];
                if (j % 4 || cl[k0 + k + 1] != j + 1 || cl[k0 + k + 2] != j + 2 || cl[k0 + k + 3] != j + 3)
                    vec_ok = false;
            }
            chunks.push_back(ci);
            // keep every chunk's element range 32-aligned in the sign bit array
            while (gcoord.size() % 32) {
                gcoord.push_back(0);
                pos.push_back(0);
            }
            while (sgnb.size() * 32 < gcoord.size()) sgnb.push_back(0);
        }
    }
    // one device allocation for the plan
    const size_t b_ch = chunks.size() * sizeof(ChunkInfoDev), b_gc = gcoord.size() * 4, b_pos = pos.size() * 2,
                 b_sg = sgnb.size() * 4, b_bp = bp.size() * 4, b_cn = cnt.size();
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t total = al(b_ch) + al(b_gc) + al(b_pos) + al(b_sg) + al(b_bp) + al(b_cn);
    CK(cudaMalloc(&H->d_cplan_mem, total));
    char* base = (char*)H->d_cplan_mem;
    size_t o = 0;
    cudaError_t perr = cudaSuccess;
    auto put = [&](const void* src, size_t b) {
        char* dst = base + o;
        if (b && perr == cudaSuccess) perr = cudaMemcpy(dst, src, b, cudaMemcpyHostToDevice);
        o += al(b);
        return (void*)dst;
    };
    ChunkedPlanDev cp{};
    cp.d = d;
    cp.m = m;
    cp.L = L;
    cp.K = K;
    cp.nchunks = (int)chunks.size();
    cp.gbins = gbins;
    cp.max_cnt = max_cnt;
    cp.vec_ok = vec_ok ? 1 : 0;
    cp.chunks = (const ChunkInfoDev*)put(chunks.data(), b_ch);
    cp.gcoord = (const int32_t*)put(gcoord.data(), b_gc);
    cp.pos = (const uint16_t*)put(pos.data(), b_pos);
    cp.sgn = (const uint32_t*)put(sgnb.data(), b_sg);
    cp.bp = (const uint32_t*)put(bp.data(), b_bp);
    cp.cnt = (const uint8_t*)put(cnt.data(), b_cn);
    CK(perr);
    H->cplan = cp;
    H->chunked = true;
    return LSH_OK;
}

// HCS slab plan (sketch_hcs.cu): slab = the d_1*d_2 contiguous inputs of one outer
// index J = (i_3..i_N); all slabs share the slab-internal bin map (h_1 + m_1 h_2,
// s_1 s_2) and add into the block g(J) of m_1*m_2 bins with sign s(J).  Built in
// addition to the generic plan, which stays the fallback for unaligned inputs.
static lsh_status build_hcs_plan(lsh_handle* H) {
    const lsh_params* p = &H->p;
    const HostTables& t = H->host;
    if (!is_hcs(p->scheme) || t.N < 3) return LSH_OK;
    const int64_t S64 = t.md[0] * t.md[1], M64 = t.mm[0] * t.mm[1];
    if (S64 > 1024 || M64 > 1024) return LSH_OK;
    const int S = (int)S64, M12 = (int)M64;
    if (!hcs_plan_supported(S, M12) || M12 % p->K != 0 || p->d % S != 0) return LSH_OK;
    if (hcs_smem_bytes(S, M12, p->m, (int)(p->d / S + p->m / M12) + 4, 0) > 232448) return LSH_OK;
    if (p->d / S > 0x7fffffff) return LSH_OK;
    std::vector<int> bin12(S);
    std::vector<uint32_t> sgn((S + 31) / 32, 0);
    for (int k = 0; k < S; ++k) {
        const int i1 = k % (int)t.md[0], i2 = k / (int)t.md[0];
        bin12[k] = t.h[0][i1] + (int)t.mm[0] * t.h[1][i2];
        if (t.s[0][i1] * t.s[1][i2] < 0) sgn[k >> 5] |= 1u << (k & 31);
    }
    // pos[q] = staged word offset (sketch_hcs.cu layout) of the coordinate at
    // bin-sorted position q; bp = bin starts in that order
    std::vector<uint16_t> bp(M12 + 1, 0), pos(S);
    for (int k = 0; k < S; ++k) bp[bin12[k] + 1]++;
    for (int b = 0; b < M12; ++b) bp[b + 1] += bp[b];
    {
        std::vector<uint16_t> cur(bp.begin(), bp.end() - 1);
        for (int k = 0; k < S; ++k) pos[cur[bin12[k]]++] = (uint16_t)((k >> 2) * 129 + (k & 3) * 32);
    }
    // bins -> 16 warps, M12/16 each, greedy by coordinate count (largest first) so the
    // per-slab gather work of the warps is balanced
    const int bpw = M12 / 16;
    std::vector<uint8_t> wbins(M12);
    {
        std::vector<int> order(M12), load(16, 0), nb(16, 0);
        for (int b = 0; b < M12; ++b) order[b] = b;
        std::stable_sort(order.begin(), order.end(),
                         [&](int a, int b) { return bp[a + 1] - bp[a] > bp[b + 1] - bp[b]; });
        for (int b : order) {
            int best = -1;
            for (int w = 0; w < 16; ++w)
                if (nb[w] < bpw && (best < 0 || load[w] < load[best])) best = w;
            wbins[best * bpw + nb[best]++] = (uint8_t)b;
            load[best] += bp[b + 1] - bp[b];
        }
    }
    const int64_t nslab = p->d / S;
    const int nblocks = p->m / M12;
    std::vector<std::vector<std::pair<uint32_t, bool>>> lists(nblocks);
    for (int64_t J = 0; J < nslab; ++J) {
        int64_t rem = J, g = 0, stride = 1;
        int sg = 1;
        for (int k = 2; k < t.N; ++k) {
            const int64_t ik = rem % t.md[k];
            rem /= t.md[k];
            g += (int64_t)t.h[k][ik] * stride;
            stride *= t.mm[k];
            sg *= t.s[k][ik];
        }
        lists[g].push_back({(uint32_t)J, sg < 0});
    }
    std::vector<uint2> ents;
    std::vector<int32_t> bfirst(nblocks);
    for (int g = 0; g < nblocks; ++g) {
        bfirst[g] = (int32_t)ents.size();
        if (lists[g].empty()) {
            ents.push_back(make_uint2(0u, (uint32_t)g | HCS_EMPTY | HCS_LAST));
            continue;
        }
        for (size_t i = 0; i < lists[g].size(); ++i) {
            uint32_t y = (uint32_t)g;
            if (lists[g][i].second) y |= HCS_NEG;
            if (i + 1 == lists[g].size()) y |= HCS_LAST;
            ents.push_back(make_uint2(lists[g][i].first, y));
        }
    }
    const size_t b_e = sizeof(uint2) * ents.size(), b_p = sizeof(uint16_t) * S, b_s = sizeof(uint32_t) * sgn.size(),
                 b_b = sizeof(uint16_t) * bp.size(), b_f = sizeof(int32_t) * bfirst.size(), b_w = wbins.size();
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    CK(cudaMalloc(&H->d_hplan_mem, al(b_e) + al(b_p) + al(b_s) + al(b_b) + al(b_f) + al(b_w)));
    char* base = (char*)H->d_hplan_mem;
    CK(cudaMemcpy(base, ents.data(), b_e, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(base + al(b_e), pos.data(), b_p, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(base + al(b_e) + al(b_p), sgn.data(), b_s, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(base + al(b_e) + al(b_p) + al(b_s), bp.data(), b_b, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(base + al(b_e) + al(b_p) + al(b_s) + al(b_b), bfirst.data(), b_f, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(base + al(b_e) + al(b_p) + al(b_s) + al(b_b) + al(b_f), wbins.data(), b_w, cudaMemcpyHostToDevice));
    HcsPlanDev hp{};
    hp.m = p->m;
    hp.K = p->K;
    hp.S = S;
    hp.M12 = M12;
    hp.nentries = (int)ents.size();
    hp.entries = (const uint2*)base;
    hp.pos = (const uint16_t*)(base + al(b_e));
    hp.sgn = (const uint32_t*)(base + al(b_e) + al(b_p));
    hp.bp = (const uint16_t*)(base + al(b_e) + al(b_p) + al(b_s));
    hp.nblocks = nblocks;
    hp.d = p->d;
    hp.bfirst = (const int32_t*)(base + al(b_e) + al(b_p) + al(b_s) + al(b_b));
    hp.wbins = (const uint8_t*)(base + al(b_e) + al(b_p) + al(b_s) + al(b_b) + al(b_f));
    H->hplan = hp;
    H->hcs = true;
    return LSH_OK;
}

static lsh_status build_plan(lsh_handle* H) {
    const lsh_params* p = &H->p;
    std::vector<int32_t> bin;
    std::vector<int8_t> sgn;
    coordinate_map(p, H->host, bin, sgn);
    const int d = (int)p->d, m = p->m;
    const int vpt = d <= 64 ? 1 : (d <= 256 ? 4 : 16);
    const int Q = 64 * vpt;
    if (d > Q || sketch_smem_bytes(Q, m, d, p->L) > 232448) return build_chunked_plan(H, bin, sgn);
    // single resident tile: bins in bin-sorted order (ascending coordinate inside a bin);
    // ent = the staged tile's word offset of each coordinate (transposed layout of sketch.cu)
    std::vector<uint32_t> bin_ptr(m + 1, 0);
    std::vector<uint16_t> ent(d);
    std::vector<uint32_t> sign_bits((d + 31) / 32, 0);
    for (int j = 0; j < d; ++j)
        if (sgn[j] < 0) sign_bits[j >> 5] |= 1u << (j & 31);
    for (int j = 0; j < d; ++j) bin_ptr[bin[j] + 1]++;
    for (int l = 0; l < m; ++l) bin_ptr[l + 1] += bin_ptr[l];
    {
        std::vector<uint32_t> cur(bin_ptr.begin(), bin_ptr.end() - 1);
        for (int j = 0; j < d; ++j) ent[cur[bin[j]]++] = (uint16_t)((j >> 2) * kSketchColWords + (j & 3) * 32);
    }
    const uint32_t ZW = (uint32_t)(Q / 4) * (uint32_t)kSketchColWords;
    int max_cnt = 0;
    // per bin: the staged words of its first two coordinates (the zero slot when
    // missing); its 3rd, 4th, ... coordinates are folded into the first one's word
    // (fold entries of the bin's table, in bin-sorted order), so the bin's sum is
    // ((x_1 + x_3) + x_4 + ...) + x_2 — the order the generic path uses too
    std::vector<uint32_t> pairs(2 * (size_t)m), fold_ptr(p->L + 1, 0), fold;
    for (int l = 0; l < m; ++l) {
        const uint32_t c = bin_ptr[l + 1] - bin_ptr[l];
        max_cnt = std::max(max_cnt, (int)c);
        const uint32_t a = c >= 1 ? ent[bin_ptr[l]] : ZW;
        const uint32_t b = c >= 2 ? ent[bin_ptr[l] + 1] : ZW;
        pairs[2 * l] = a * 4u;       // byte offsets inside the staged tile
        pairs[2 * l + 1] = b * 4u;
        for (uint32_t j = 2; j < c; ++j) fold.push_back((a << 16) | ent[bin_ptr[l] + j]);
        fold_ptr[l / p->K + 1] = (uint32_t)fold.size();
    }
    for (int t = 0; t < p->L; ++t) fold_ptr[t + 1] = std::max(fold_ptr[t + 1], fold_ptr[t]);
    std::vector<uint32_t> fold_all(fold_ptr.begin(), fold_ptr.end());
    fold_all.insert(fold_all.end(), fold.begin(), fold.end());
    CK(cudaMalloc(&H->d_entries, sizeof(uint16_t) * std::max(1, d)));
    CK(cudaMalloc(&H->d_binptr, sizeof(uint32_t) * bin_ptr.size()));
    CK(cudaMalloc(&H->d_signs, sizeof(uint32_t) * sign_bits.size()));
    CK(cudaMalloc(&H->d_pairs, sizeof(uint32_t) * 2 * (size_t)m));
    CK(cudaMalloc(&H->d_fold, sizeof(uint32_t) * fold_all.size()));
    CK(cudaMemcpy(H->d_entries, ent.data(), sizeof(uint16_t) * d, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(H->d_binptr, bin_ptr.data(), sizeof(uint32_t) * bin_ptr.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(H->d_signs, sign_bits.data(), sizeof(uint32_t) * sign_bits.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(H->d_pairs, pairs.data(), sizeof(uint32_t) * 2 * (size_t)m, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(H->d_fold, fold_all.data(), sizeof(uint32_t) * fold_all.size(), cudaMemcpyHostToDevice));
    H->plan = SketchPlanDev{d, m, p->L, p->K, Q, vpt, 1, max_cnt, H->d_entries, H->d_binptr, H->d_signs,
                            H->d_pairs, H->d_fold, H->d_fold + p->L + 1, (int)fold.size()};
    return LSH_OK;
}

static void free_handle(lsh_handle* H) {
    if (!H) return;
    cudaFree(H->d_entries);
    cudaFree(H->d_binptr);
    cudaFree(H->d_cplan_mem);
    cudaFree(H->d_hplan_mem);
    cudaFree(H->d_signs);
    cudaFree(H->d_pairs);
    cudaFree(H->d_fold);
    cudaFree(H->d_coff);
    cudaFree(H->d_R);
    cudaFree(H->d_Rpad);
    cudaFree(H->d_flags);
    for (auto x : H->d_h) cudaFree(x);
    for (auto x : H->d_s) cudaFree(x);
    cudaFree(H->d_b);
    delete H;
}

extern "C" lsh_status lsh_create(const lsh_params* p, lsh_handle** out) {
    if (!out) return LSH_ESTATE;
    *out = nullptr;
    lsh_status st = validate(p);
    if (st != LSH_OK) return st;
    lsh_handle* H = new lsh_handle();
    H->p = *p;
    H->device = p->device;
    auto fail = [&](lsh_status s) {
        free_handle(H);
        return s;
    };
    cudaError_t e = cudaSetDevice(p->device);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaSetDevice"));
    cudaDeviceGetAttribute(&H->num_sms, cudaDevAttrMultiProcessorCount, p->device);
    {
        // Scratch and index buffers come from the device's stream-ordered pool; keep freed
        // memory cached in the pool instead of unmapping it at every synchronisation.
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, p->device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    try {
        draw(p, H->host, true);
    } catch (...) {
        return fail(LSH_ENOMEM);
    }
    H->key_width = is_e2lsh(p->scheme) ? 64 : p->K;
    const int m = p->m;
    // offsets folded with w: c_off[l] = b_l / w; c_scale = sqrt(m)/w (CS/HCS) or 1/w (dense)
    std::vector<float> coff(m);
    for (int l = 0; l < m; ++l) coff[l] = (float)((double)H->host.b[l] / (double)p->w);
    const double scale = is_dense(p->scheme) ? 1.0
                         : is_per_table(p)   ? (double)sqrtf((float)p->K)   // reading C3: sketch size K
                                             : (double)sqrtf((float)m);
    H->disc.e2lsh = is_e2lsh(p->scheme) ? 1 : 0;
    H->disc.c_scale = (float)(scale / (double)p->w);
    if ((e = cudaMalloc(&H->d_coff, sizeof(float) * m)) != cudaSuccess) return fail(cuda_fail(e, "malloc"));
    if ((e = cudaMemcpy(H->d_coff, coff.data(), sizeof(float) * m, cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(cuda_fail(e, "memcpy"));
    // [0] sticky device status (overflow), [1] grouping-path hint (group.cu: launch_group)
    if ((e = cudaMalloc(&H->d_flags, 2 * sizeof(int))) != cudaSuccess) return fail(cuda_fail(e, "malloc"));
    if ((e = cudaMemset(H->d_flags, 0, 2 * sizeof(int))) != cudaSuccess) return fail(cuda_fail(e, "memset"));
    H->disc.c_off = H->d_coff;
    H->disc.flags = H->d_flags;
    if ((e = cudaMalloc(&H->d_b, sizeof(float) * m)) != cudaSuccess) return fail(cuda_fail(e, "malloc"));
    if ((e = cudaMemcpy(H->d_b, H->host.b.data(), sizeof(float) * m, cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(cuda_fail(e, "memcpy b"));
    if (uses_R(p)) {
        const size_t bytes = sizeof(uint16_t) * H->host.R.size();
        if ((e = cudaMalloc(&H->d_R, bytes)) != cudaSuccess) return fail(cuda_fail(e, "malloc R"));
        if ((e = cudaMemcpy(H->d_R, H->host.R.data(), bytes, cudaMemcpyHostToDevice)) != cudaSuccess)
            return fail(cuda_fail(e, "memcpy R"));
        H->d_pad = (int)((p->d + 63) / 64 * 64);
        const size_t pbytes = sizeof(uint16_t) * (size_t)m * H->d_pad;
        if ((e = cudaMalloc(&H->d_Rpad, pbytes)) != cudaSuccess) return fail(cuda_fail(e, "malloc Rpad"));
        if ((e = cudaMemset(H->d_Rpad, 0, pbytes)) != cudaSuccess) return fail(cuda_fail(e, "memset Rpad"));
        if ((e = cudaMemcpy2D(H->d_Rpad, sizeof(uint16_t) * H->d_pad, H->d_R, sizeof(uint16_t) * p->d,
                              sizeof(uint16_t) * p->d, m, cudaMemcpyDeviceToDevice)) != cudaSuccess)
            return fail(cuda_fail(e, "pad R"));
    } else {
        for (int k = 0; k < H->host.N; ++k) {
            int32_t *dh = nullptr, *ds = nullptr;
            const size_t bytes = sizeof(int32_t) * H->host.h[k].size();
            if ((e = cudaMalloc(&dh, bytes)) != cudaSuccess) return fail(cuda_fail(e, "malloc h"));
            H->d_h.push_back(dh);
            if ((e = cudaMalloc(&ds, bytes)) != cudaSuccess) return fail(cuda_fail(e, "malloc s"));
            H->d_s.push_back(ds);
            if ((e = cudaMemcpy(dh, H->host.h[k].data(), bytes, cudaMemcpyHostToDevice)) != cudaSuccess ||
                (e = cudaMemcpy(ds, H->host.s[k].data(), bytes, cudaMemcpyHostToDevice)) != cudaSuccess)
                return fail(cuda_fail(e, "memcpy h/s"));
        }
        try {
            st = build_plan(H);
            if (st == LSH_OK) st = build_hcs_plan(H);
        } catch (...) {
            st = LSH_ENOMEM;
        }
        if (st != LSH_OK) return fail(st);
    }
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return fail(cuda_fail(e, "create sync"));
    *out = H;
    return LSH_OK;
}

extern "C" void lsh_destroy(lsh_handle* h) { free_handle(h); }

extern "C" lsh_status lsh_check(const lsh_handle* h) {
    if (!h) return LSH_ESTATE;
    CK(cudaSetDevice(h->device));
    CK(cudaDeviceSynchronize());
    int flags = 0;
    CK(cudaMemcpy(&flags, h->d_flags, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemset(h->d_flags, 0, sizeof(int)));
    if (flags & 3) return LSH_EOVERFLOW;
    if (flags & 4) return LSH_EUNSUPPORTED;
    return LSH_OK;
}

extern "C" lsh_status lsh_group_path(const lsh_handle* h, int32_t* path) {
    if (!h || !path) return LSH_ESTATE;
    CK(cudaSetDevice(h->device));
    CK(cudaDeviceSynchronize());
    int flags[2] = {0, 0};
    CK(cudaMemcpy(flags, h->d_flags, sizeof(flags), cudaMemcpyDeviceToHost));
    *path = flags[1];
    return LSH_OK;
}

// ---------------------------------------------------------------------------
// hashing
// ---------------------------------------------------------------------------
static lsh_status hash_impl(const lsh_handle* H, const float* X, int64_t n, int64_t ld, HashOut out, cudaStream_t s,
                            const char* tname = "sketch") {
    const lsh_params& p = H->p;
    if (out.bits && !is_e2lsh(p.scheme)) {
        CK(cudaMemsetAsync(out.bits, 0, sizeof(uint32_t) * (size_t)n * ((p.m + 31) / 32), s));
    }
    if (out.codes && !is_e2lsh(p.scheme)) out.codes = nullptr;
    if (out.bits && is_e2lsh(p.scheme)) out.bits = nullptr;
    if (n == 0) return LSH_OK;
    if (uses_R(&p)) {
        static const bool unfused = getenv("LSH_DENSE_UNFUSED") && getenv("LSH_DENSE_UNFUSED")[0] == '1';
        cudaError_t e;
        if (!unfused && out.keys && !out.codes && !out.bits && !out.proj &&
            dense_tc_fused_keys_ok(p.m, p.K)) {
            // keys straight from the accumulators (fused epilogue): no [n][m] projection in HBM
            const int64_t rows = std::min<int64_t>(n, (int64_t)dense_tc_rows_per_batch(H->d_pad));
            uint16_t* A = nullptr;
            CK(cudaMallocAsync((void**)&A, sizeof(uint16_t) * (size_t)rows * 3 * H->d_pad, s));
            const std::string gname = std::string(tname) == "sketch" ? "dense_gemm" : "dense_gemm_query";
            timing_begin(gname.c_str(), s);
            e = launch_dense_tc(X, n, ld, (int)p.d, H->d_Rpad, p.m, H->d_pad, A, rows, nullptr, s, out.keys, p.K,
                                &H->disc);
            timing_end(gname.c_str(), s);
            CK(cudaFreeAsync(A, s));
            if (e != cudaSuccess) return cuda_fail(e, "dense_gemm");
            return LSH_OK;
        }
        float* Y = out.proj;
        if (!Y) CK(cudaMallocAsync((void**)&Y, sizeof(float) * (size_t)n * p.m, s));
        {
            const int64_t rows = std::min<int64_t>(n, (int64_t)dense_tc_rows_per_batch(H->d_pad));
            uint16_t* A = nullptr;
            CK(cudaMallocAsync((void**)&A, sizeof(uint16_t) * (size_t)rows * 3 * H->d_pad, s));
            const std::string gname = std::string(tname) == "sketch" ? "dense_gemm" : "dense_gemm_query";
            timing_begin(gname.c_str(), s);
            e = launch_dense_tc(X, n, ld, (int)p.d, H->d_Rpad, p.m, H->d_pad, A, rows, Y, s);
            timing_end(gname.c_str(), s);
            CK(cudaFreeAsync(A, s));
        }
        if (e != cudaSuccess) return cuda_fail(e, "dense_gemm");
        timing_begin("keys_from_proj", s);
        e = launch_keys_from_proj(Y, n, p.m, p.L, p.K, H->disc, out, s);
        count_launch();
        timing_end("keys_from_proj", s);
        if (e != cudaSuccess) return cuda_fail(e, "keys_from_proj");
        if (!out.proj) CK(cudaFreeAsync(Y, s));
        return LSH_OK;
    }
    if (!H->sketch_ok && !H->hcs) return LSH_EUNSUPPORTED;
    timing_begin(tname, s);
    const bool hcs_vec = H->hcs && (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0) &&
                         !(getenv("LSH_NO_HCS_SLAB") && getenv("LSH_NO_HCS_SLAB")[0] == '1');
    if (!hcs_vec && !H->sketch_ok) {
        timing_end(tname, s);
        return LSH_EUNSUPPORTED;
    }
    cudaError_t e = hcs_vec      ? launch_sketch_hcs(H->hplan, H->disc, X, n, ld, out, H->num_sms, s)
                    : H->chunked ? launch_sketch_chunked(H->cplan, H->disc, X, n, ld, out, H->num_sms, s)
                                 : launch_sketch(H->plan, H->disc, X, n, ld, out, H->num_sms, s);
    count_launch();
    timing_end(tname, s);
    if (e != cudaSuccess) return cuda_fail(e, "sketch");
    return LSH_OK;
}

extern "C" lsh_status lsh_hash(const lsh_handle* h, const float* X, int64_t n, int64_t ld, uint64_t* keys,
                               int32_t* codes, uint32_t* bits, float* proj, void* stream) {
    if (!h) return LSH_ESTATE;
    if (n < 0 || ld < h->p.d) return LSH_EDIM;
    if (n > 0 && !X) return LSH_EDIM;
    CK(cudaSetDevice(h->device));
    return hash_impl(h, X, n, ld, HashOut{keys, codes, bits, proj}, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// index
// ---------------------------------------------------------------------------
static lsh_status alloc_index(const lsh_handle* H, int64_t n, cudaStream_t s, lsh_index** out) {
    lsh_index* I = new lsh_index();
    I->h = H;
    I->n = n;
    I->stream = s;
    I->L = H->p.L;
    const int L = I->L;
    const size_t b_ids = sizeof(uint32_t) * (size_t)L * n;
    const size_t b_uk = sizeof(uint64_t) * (size_t)L * n;
    const size_t b_off = sizeof(uint32_t) * (size_t)L * (n + 1);
    const size_t b_nb = sizeof(uint32_t) * L;
    const size_t total = b_uk + b_ids + b_off + b_nb + 64;
    cudaError_t e = cudaMallocAsync(&I->mem, total, s);
    if (e != cudaSuccess) {
        delete I;
        return cuda_fail(e, "index alloc");
    }
    char* base = (char*)I->mem;
    I->dev.ukeys = (uint64_t*)base;
    I->dev.ids = (uint32_t*)(base + b_uk);
    I->dev.offs = (uint32_t*)(base + b_uk + b_ids);
    I->dev.nb = (uint32_t*)(base + b_uk + b_ids + b_off);
    cudaEventCreateWithFlags(&I->done, cudaEventDisableTiming);
    *out = I;
    return LSH_OK;
}

static lsh_status group_impl(const lsh_handle* H, const uint64_t* keys, uint64_t* keys_scratch, int64_t n,
                             int64_t id_base, lsh_index* I, cudaStream_t s) {
    // keys_scratch: a dead [L][n] u64 buffer (the hashed keys of lsh_build_index, fully
    // consumed by the L1 scatter before the per-bin kernel runs) reused as [L][2n] u32
    // permutation scratch; nullptr = allocate it.
    const int L = H->p.L;
    GroupScratch sc{};
    const size_t nb1 = (size_t)group_bins(n, H->key_width);
    // L1 output: [L][n] (histogram path) or the fixed-capacity layout [L][nb1][cap]
    const size_t slots = group_key_slots(n, H->key_width);
    const size_t b_keys = sizeof(uint64_t) * (size_t)L * slots;
    const size_t b_ids = sizeof(uint32_t) * (size_t)L * slots;
    const size_t b_hist = sizeof(uint32_t) * (size_t)L * std::max<size_t>(group_hist_words(n, H->key_width), 1);
    const size_t b_tot = sizeof(uint32_t) * (size_t)L * nb1;
    const size_t b_bs = sizeof(uint32_t) * (size_t)L * (nb1 + 1);
    const size_t b_st = sizeof(unsigned long long) * (size_t)L * std::max<size_t>(nb1, (size_t)group_rle_chunks(n));
    const bool own_perm = (keys_scratch == nullptr);
    const size_t b_perm = own_perm ? b_keys : 0;
    const size_t b_vm = sizeof(unsigned long long) * 2 * (size_t)L;
    const size_t b_spec = group_spec_bytes() * 2 * (size_t)L;
    const size_t b_cb = sizeof(uint32_t) * ((size_t)L * nb1 + 3);   // big-bin count, g2a ticket, overflow, big-bin list
    void* mem = nullptr;
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t total = al(b_keys) + al(b_ids) + al(b_hist) + al(b_tot) + al(b_bs) + al(b_st) + al(b_perm) + al(b_vm) +
                         al(b_spec) + al(b_cb);
    if (n > 0) CK(cudaMallocAsync(&mem, total, s));
    char* p = (char*)mem;
    auto take = [&](size_t b) {
        char* r = p;
        p += al(b);
        return r;
    };
    if (n > 0) {
        sc.keys_a = (uint64_t*)take(b_keys);
        sc.ids_a = (uint32_t*)take(b_ids);
        sc.hist = (uint32_t*)take(b_hist);
        sc.tot = (uint32_t*)take(b_tot);
        sc.binstart = (uint32_t*)take(b_bs);
        sc.state = (unsigned long long*)take(b_st);
        sc.perm = own_perm ? (uint32_t*)take(b_perm) : (uint32_t*)keys_scratch;
        sc.vmask = (unsigned long long*)take(b_vm);
        sc.spec = take(b_spec);
        sc.bigcount = (uint32_t*)take(b_cb);
        sc.biglist = sc.bigcount + 3;
    }
    sc.num_sms = H->num_sms;
    cudaError_t e = launch_group(keys, n, L, (uint32_t)id_base, H->key_width, sc, I->dev, H->d_flags, s);
    if (e != cudaSuccess) return cuda_fail(e, "group");
    if (mem) CK(cudaFreeAsync(mem, s));
    CK(cudaEventRecord(I->done, s));
    return LSH_OK;
}

extern "C" lsh_status lsh_group_keys(const lsh_handle* h, const uint64_t* keys, int64_t n, int64_t id_base,
                                     lsh_index** out, void* stream) {
    if (!h || !out) return LSH_ESTATE;
    if (n < 0 || id_base < 0 || id_base + n > (1ll << 32) - 1) return LSH_EDIM;
    CK(cudaSetDevice(h->device));
    cudaStream_t s = (cudaStream_t)stream;
    lsh_index* I = nullptr;
    lsh_status st = alloc_index(h, n, s, &I);
    if (st != LSH_OK) return st;
    I->id_base = id_base;
    st = group_impl(h, keys, nullptr, n, id_base, I, s);
    if (st != LSH_OK) {
        lsh_index_destroy(I);
        return st;
    }
    *out = I;
    return LSH_OK;
}

extern "C" lsh_status lsh_build_index(const lsh_handle* h, const float* X, int64_t n, int64_t ld, int64_t id_base,
                                      lsh_index** out, void* stream) {
    if (!h || !out) return LSH_ESTATE;
    if (n < 0 || ld < h->p.d || id_base < 0 || id_base + n > (1ll << 32) - 1) return LSH_EDIM;
    if (n > 0 && !X) return LSH_EDIM;
    CK(cudaSetDevice(h->device));
    cudaStream_t s = (cudaStream_t)stream;
    lsh_index* I = nullptr;
    lsh_status st = alloc_index(h, n, s, &I);
    if (st != LSH_OK) return st;
    uint64_t* keys = nullptr;
    if (n > 0) {
        cudaError_t e = cudaMallocAsync((void**)&keys, sizeof(uint64_t) * (size_t)h->p.L * n, s);
        if (e != cudaSuccess) {
            lsh_index_destroy(I);
            return cuda_fail(e, "keys alloc");
        }
    }
    I->id_base = id_base;
    st = hash_impl(h, X, n, ld, HashOut{keys, nullptr, nullptr, nullptr}, s);
    if (st == LSH_OK) st = group_impl(h, keys, keys, n, id_base, I, s);
    if (keys) cudaFreeAsync(keys, s);
    if (st != LSH_OK) {
        lsh_index_destroy(I);
        return st;
    }
    *out = I;
    return LSH_OK;
}

extern "C" lsh_status lsh_index_view(const lsh_index* idx, int32_t t, const uint32_t** ids, const uint64_t** ukeys,
                                     const uint32_t** offs, int64_t* nb) {
    if (!idx) return LSH_ESTATE;
    if (t < 0 || t >= idx->L) return LSH_EDIM;
    CK(cudaEventSynchronize(idx->done));
    uint32_t nbv = 0;
    CK(cudaMemcpy(&nbv, idx->dev.nb + t, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    const int64_t n = idx->n;
    if (ids) *ids = idx->dev.ids + (int64_t)t * n;
    if (ukeys) *ukeys = idx->dev.ukeys + (int64_t)t * n;
    if (offs) *offs = idx->dev.offs + (int64_t)t * (n + 1);
    if (nb) *nb = nbv;
    return LSH_OK;
}

extern "C" int64_t lsh_index_size(const lsh_index* idx) { return idx ? idx->n : -1; }

extern "C" void lsh_index_destroy(lsh_index* idx) {
    if (!idx) return;
    cudaSetDevice(idx->h->device);
    {
        // the stream-ordered free runs after every recorded reader on other streams
        std::lock_guard<std::mutex> g(idx->use_mu);
        for (auto& u : idx->uses) {
            cudaStreamWaitEvent(idx->stream, u.second, 0);
            cudaEventDestroy(u.second);
        }
        idx->uses.clear();
    }
    if (idx->mem) cudaFreeAsync(idx->mem, idx->stream);
    if (idx->done) cudaEventDestroy(idx->done);
    delete idx;
}

extern "C" lsh_status lsh_query_buckets(const lsh_handle* h, const lsh_index* idx, const float* Q, int64_t nq,
                                        int64_t ld, int64_t* begin, int64_t* end, void* stream) {
    if (!h || !idx || idx->h->p.L != h->p.L) return LSH_ESTATE;
    if (nq < 0 || ld < h->p.d) return LSH_EDIM;
    if (nq == 0) return LSH_OK;
    if (!Q || !begin || !end) return LSH_EDIM;
    CK(cudaSetDevice(h->device));
    cudaStream_t s = (cudaStream_t)stream;
    uint64_t* qk = nullptr;
    CK(cudaMallocAsync((void**)&qk, sizeof(uint64_t) * (size_t)h->p.L * nq, s));
    lsh_status st = hash_impl(h, Q, nq, ld, HashOut{qk, nullptr, nullptr, nullptr}, s, "sketch_query");
    if (st == LSH_OK) {
        CK(index_acquire(idx, s));
        timing_begin("lookup", s);
        cudaError_t e = launch_lookup(qk, nq, h->p.L, idx->n, idx->dev, begin, end, h->key_width == 64, s);
        count_launch();
        timing_end("lookup", s);
        if (e != cudaSuccess) st = cuda_fail(e, "lookup");
        index_release(idx, s);
    }
    cudaFreeAsync(qk, s);
    return st;
}

extern "C" lsh_status lsh_query_knn(const lsh_handle* h, const lsh_index* idx, const float* X, int64_t ldx,
                                    const float* Q, int64_t nq, int64_t ldq, int32_t k, int32_t max_cand,
                                    int64_t* out_ids, float* out_score, int32_t* out_ncand, void* stream) {
    if (!h || !idx || idx->h->p.L != h->p.L) return LSH_ESTATE;
    if (k < 1 || max_cand < k || max_cand > 8192) return LSH_EINVAL;
    if (nq < 0 || ldq < h->p.d || ldx < h->p.d) return LSH_EDIM;
    if (nq == 0) return LSH_OK;
    if (!X || !Q || !out_ids || !out_score) return LSH_EDIM;
    CK(cudaSetDevice(h->device));
    cudaStream_t s = (cudaStream_t)stream;
    const int L = h->p.L;
    int64_t* be = nullptr;
    CK(cudaMallocAsync((void**)&be, sizeof(int64_t) * 2 * (size_t)nq * L, s));
    lsh_status st = lsh_query_buckets(h, idx, Q, nq, ldq, be, be + (size_t)nq * L, stream);
    if (st == LSH_OK) {
        CK(index_acquire(idx, s));
        timing_begin("knn", s);
        cudaError_t e = launch_knn(idx->dev, idx->n, L, (uint32_t)idx->id_base, be, be + (size_t)nq * L, X, ldx,
                                   (int)h->p.d, Q, ldq, nq, k, max_cand, is_e2lsh(h->p.scheme) ? 0 : 1, out_ids,
                                   out_score, out_ncand, s);
        count_launch();
        timing_end("knn", s);
        if (e != cudaSuccess) st = cuda_fail(e, "knn");
        index_release(idx, s);
    }
    cudaFreeAsync(be, s);
    return st;
}

extern "C" lsh_status lsh_index_counts(const lsh_index* idx, int32_t B, uint32_t* counts, void* stream) {
    if (!idx) return LSH_ESTATE;
    if (B < 1 || B > 20 || !counts) return LSH_EDIM;
    CK(cudaSetDevice(idx->h->device));
    cudaStream_t s = (cudaStream_t)stream;
    CK(index_acquire(idx, s));
    timing_begin("counts", s);
    cudaError_t e = launch_counts(idx->dev, idx->n, idx->L, idx->h->key_width, B, counts, s);
    count_launch();
    timing_end("counts", s);
    index_release(idx, s);
    if (e != cudaSuccess) return cuda_fail(e, "counts");
    return LSH_OK;
}

extern "C" lsh_status lsh_global_offsets(const uint32_t* all_counts, int32_t G, int32_t rank, int32_t L, int32_t B,
                                        int64_t* offsets, void* stream) {
    if (G < 1 || rank < 0 || rank >= G || L < 1 || B < 1 || B > 20 || !all_counts || !offsets) return LSH_EDIM;
    cudaStream_t s = (cudaStream_t)stream;
    timing_begin("global_offsets", s);
    cudaError_t e = launch_global_offsets(all_counts, G, rank, L, B, offsets, s);
    count_launch();
    timing_end("global_offsets", s);
    if (e != cudaSuccess) return cuda_fail(e, "global_offsets");
    return LSH_OK;
}

extern "C" lsh_status lsh_query_global_runs(const int64_t* all_ranges, int32_t G, int32_t rank, int64_t M,
                                           int64_t* gbegin, int64_t* gtotal, void* stream) {
    if (G < 1 || rank < 0 || rank >= G || M < 0 || (M > 0 && (!all_ranges || !gbegin))) return LSH_EDIM;
    cudaStream_t s = (cudaStream_t)stream;
    timing_begin("query_runs", s);
    cudaError_t e = launch_query_runs(all_ranges, G, rank, M, gbegin, gtotal, s);
    if (M > 0) count_launch();
    timing_end("query_runs", s);
    if (e != cudaSuccess) return cuda_fail(e, "query_runs");
    return LSH_OK;
}

// ---------------------------------------------------------------------------
// parameter export
// ---------------------------------------------------------------------------
static lsh_status export_from(const lsh_params* p, const HostTables& t, int32_t what, int32_t mode, void* buf,
                              size_t* bytes) {
    if (!bytes) return LSH_EDIM;
    std::vector<unsigned char> out;
    auto put = [&](const void* src, size_t nb) {
        out.resize(nb);
        if (nb) std::memcpy(out.data(), src, nb);
    };
    switch (what) {
        case LSH_EXPORT_BUCKET:
        case LSH_EXPORT_SIGN:
        case LSH_EXPORT_COEFFS: {
            // per-table families: `mode` = table index
            if (is_dense(p->scheme) || mode < 0 || mode >= t.N) return LSH_EINVAL;
            if (what == LSH_EXPORT_BUCKET) put(t.h[mode].data(), t.h[mode].size() * 4);
            else if (what == LSH_EXPORT_SIGN) put(t.s[mode].data(), t.s[mode].size() * 4);
            else {
                uint64_t c[4] = {t.fb[mode].a, t.fb[mode].b, t.fs[mode].a, t.fs[mode].b};
                put(c, sizeof(c));
            }
            break;
        }
        case LSH_EXPORT_OFFSETS: put(t.b.data(), t.b.size() * 4); break;
        case LSH_EXPORT_GAUSSIAN:
            if (!uses_R(p)) return LSH_EINVAL;
            put(t.R.data(), t.R.size() * 2);
            break;
        case LSH_EXPORT_COORD: {
            if (is_dense(p->scheme) || is_per_table(p)) return LSH_EINVAL;
            std::vector<int32_t> bin;
            std::vector<int8_t> sg;
            coordinate_map(p, t, bin, sg);
            std::vector<int32_t> v(2 * p->d);
            for (int64_t j = 0; j < p->d; ++j) {
                v[j] = bin[j];
                v[p->d + j] = sg[j];
            }
            put(v.data(), v.size() * 4);
            break;
        }
        default: return LSH_EINVAL;
    }
    if (!buf || *bytes < out.size()) {
        *bytes = out.size();
        return LSH_EDIM;
    }
    *bytes = out.size();
    if (!out.empty()) std::memcpy(buf, out.data(), out.size());
    return LSH_OK;
}

extern "C" lsh_status lsh_export_host(const lsh_params* p, int32_t what, int32_t mode, void* host_buf,
                                      size_t* bytes) {
    lsh_status st = validate(p);
    if (st != LSH_OK) return st;
    try {
        HostTables t;
        draw(p, t, what == LSH_EXPORT_GAUSSIAN);
        return export_from(p, t, what, mode, host_buf, bytes);
    } catch (...) {
        return LSH_ENOMEM;
    }
}

extern "C" lsh_status lsh_get_params(const lsh_handle* h, int32_t what, int32_t mode, void* host_buf,
                                     size_t* bytes) {
    if (!h) return LSH_ESTATE;
    CK(cudaSetDevice(h->device));
    // Read back the DEVICE copies so the check covers what the kernels use.
    HostTables t = h->host;
    if (what == LSH_EXPORT_OFFSETS) CK(cudaMemcpy(t.b.data(), h->d_b, 4 * t.b.size(), cudaMemcpyDeviceToHost));
    if (what == LSH_EXPORT_GAUSSIAN && h->d_R)
        CK(cudaMemcpy(t.R.data(), h->d_R, 2 * t.R.size(), cudaMemcpyDeviceToHost));
    if ((what == LSH_EXPORT_BUCKET || what == LSH_EXPORT_SIGN) && mode >= 0 && mode < (int)h->d_h.size()) {
        CK(cudaMemcpy(t.h[mode].data(), h->d_h[mode], 4 * t.h[mode].size(), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(t.s[mode].data(), h->d_s[mode], 4 * t.s[mode].size(), cudaMemcpyDeviceToHost));
    }
    return export_from(&h->p, t, what, mode, host_buf, bytes);
}
