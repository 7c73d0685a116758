// params.hpp — host-side parameter draw of the hashers (C++17, no CUDA).
//
// Independent implementation of DESIGN.md readings R1-R4:
//   R1 stream(seed, label) = SplitMix64 seeded with seed ^ FNV-1a-64(label)
//   R2 2-wise family over P = 2^61-1: a = 1 + next() % (P-1), b = next() % P,
//      eval(i) = ((a*(i+1) + b) mod P) mod range; sign family = range 2,
//      parity 0 -> +1, parity 1 -> -1
//   R3 offsets b_l = fp32(w * (next() >> 11) * 2^-53), clamped below w
//   R4 Gaussian R: Box-Muller on pairs, row-major, rounded to bf16 (RNE)
// The paper only requires "2-wise independent random hash functions" (PAPER.md:207,
// :210), Gaussian rows and b uniform in [0, w].
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace lshb {

constexpr uint64_t kFnvOffset = 0xcbf29ce484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001b3ull;
constexpr uint64_t kP61 = (1ull << 61) - 1;

inline uint64_t fnv1a64_bytes(const std::string& s) {
    uint64_t h = kFnvOffset;
    for (unsigned char c : s) {
        h ^= c;
        h *= kFnvPrime;
    }
    return h;
}

inline uint64_t splitmix_finalise(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// SplitMix64 sub-stream for one label.  State k (0-based) is seedmix + (k+1)*gamma,
// so the stream can be entered at any position (used to parallelise R generation).
struct Stream {
    uint64_t state;
    Stream(uint64_t seed, const std::string& label) : state(seed ^ fnv1a64_bytes(label)) {}
    uint64_t next() {
        state += 0x9e3779b97f4a7c15ull;
        return splitmix_finalise(state);
    }
    double unit53() { return (double)(next() >> 11) * 0x1.0p-53; }
};

struct TwoWise {
    uint64_t a = 0, b = 0, range = 1;
    TwoWise() = default;
    TwoWise(Stream& st, uint64_t rng_range) : range(rng_range) {
        a = 1 + st.next() % (kP61 - 1);
        b = st.next() % kP61;
    }
    uint64_t eval(uint64_t i) const {
        unsigned __int128 v = (unsigned __int128)a * (unsigned __int128)(i + 1) + b;
        return (uint64_t)(v % kP61) % range;
    }
};

// `prefix` = "table{t}/" for the per-table families (NEXT-2, reading C3).
inline std::string mode_label(int k, const char* what, const std::string& prefix = "") {
    return prefix + "mode" + std::to_string(k) + "/" + what;
}

inline TwoWise bucket_family(uint64_t seed, int k, uint64_t m_k, const std::string& prefix = "") {
    Stream st(seed, mode_label(k, "bucket", prefix));
    return TwoWise(st, m_k);
}
inline TwoWise sign_family(uint64_t seed, int k, const std::string& prefix = "") {
    Stream st(seed, mode_label(k, "sign", prefix));
    return TwoWise(st, 2);
}

inline void offsets(uint64_t seed, int m, float w, std::vector<float>& out, const std::string& prefix = "") {
    Stream st(seed, prefix + "offsets");
    out.resize(m);
    for (int l = 0; l < m; ++l) {
        double u = st.unit53();
        float b = (float)((double)w * u);
        if (!(b < w)) b = std::nextafterf(w, 0.0f);
        out[l] = b;
    }
}

// Round a double to bf16 with round-to-nearest-even, returning the 16-bit pattern.
inline uint16_t double_to_bf16_bits(double x) {
    uint64_t bits;
    std::memcpy(&bits, &x, 8);
    if (x == 0.0) return (uint16_t)((bits >> 48) & 0x8000);
    const int drop = 52 - 7;
    uint64_t lsb = (bits >> drop) & 1;
    bits += ((1ull << (drop - 1)) - 1) + lsb;
    bits = (bits >> drop) << drop;           // double holding the rounded value
    double r;
    std::memcpy(&r, &bits, 8);
    float f = (float)r;                      // exact: 8 significant bits
    uint32_t fb;
    std::memcpy(&fb, &f, 4);
    return (uint16_t)(fb >> 16);
}

inline float bf16_bits_to_float(uint16_t b) {
    uint32_t fb = (uint32_t)b << 16;
    float f;
    std::memcpy(&f, &fb, 4);
    return f;
}

// Box-Muller Gaussians, pair p of the stream fills R[2p], R[2p+1] (row-major).
// Pair p consumes outputs 2p and 2p+1 of the stream, so ranges can be generated
// independently.
inline void gaussian_range(uint64_t seed, int64_t total, int64_t pair_lo, int64_t pair_hi, uint16_t* out) {
    Stream base(seed, "gaussian");
    for (int64_t pr = pair_lo; pr < pair_hi; ++pr) {
        Stream st = base;
        st.state += (uint64_t)(2 * pr) * 0x9e3779b97f4a7c15ull;
        double u1 = 1.0 - st.unit53();
        double u2 = st.unit53();
        double rho = std::sqrt(-2.0 * std::log(u1));
        double z0 = rho * std::cos(2.0 * M_PI * u2);
        double z1 = rho * std::sin(2.0 * M_PI * u2);
        int64_t k = 2 * pr;
        out[k] = double_to_bf16_bits(z0);
        if (k + 1 < total) out[k + 1] = double_to_bf16_bits(z1);
    }
}

}  // namespace lshb
