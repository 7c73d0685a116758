// sketch_fast.cu — the keys-only K1 hot paths (K = 8 and 16, 128-bit staging),
// instantiated apart from sketch.cu so the two compile in parallel.  Kernel body:
// sketch_kernel.cuh.
#include "sketch_kernel.cuh"

namespace lshb {

template <int Q4>
static cudaError_t launch_fast_q(const SketchPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n,
                                 int64_t ld, HashOut out, int num_sms, cudaStream_t s) {
    const bool e2 = dz.e2lsh != 0;
    if (plan.K == 16)
        return e2 ? sk::launch_t<Q4, true, 16, true>(plan, dz, X, n, ld, out, num_sms, s)
                  : sk::launch_t<Q4, true, 16, false>(plan, dz, X, n, ld, out, num_sms, s);
    return e2 ? sk::launch_t<Q4, true, 8, true>(plan, dz, X, n, ld, out, num_sms, s)
              : sk::launch_t<Q4, true, 8, false>(plan, dz, X, n, ld, out, num_sms, s);
}

cudaError_t launch_sketch_fast(const SketchPlanDev& plan, const DiscretizeDev& dz, const float* X, int64_t n,
                               int64_t ld, HashOut out, int num_sms, cudaStream_t s) {
    switch (plan.vpt) {
        case 1: return launch_fast_q<16>(plan, dz, X, n, ld, out, num_sms, s);
        case 4: return launch_fast_q<64>(plan, dz, X, n, ld, out, num_sms, s);
        case 16: return launch_fast_q<256>(plan, dz, X, n, ld, out, num_sms, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lshb
