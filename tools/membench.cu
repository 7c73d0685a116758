// Read-pattern microbenchmark (diagnostic, not product code): which access shapes
// stream at HBM speed on B200?  X = n rows x d floats (row-major), summed per CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/membench tools/membench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void contiguous(const float4* __restrict__ x, size_t n4, float* out) {
    float s = 0.f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float4 v = __ldcs(x + i);
        s += v.x + v.y + v.z + v.w;
    }
    if (s == 12345.f) out[0] = s;
}

// CTA: tiles of 32 rows; per tile, slabs of W floats (all rows), slab order rotated
// by `rot` per tile.  Lanes along columns (coalesced W*4 bytes per row).
__global__ void slabs(const float* __restrict__ X, int64_t n, int64_t d, int W, int rot, float* out) {
    const int64_t ntiles = n / 32;
    const int nslab = (int)(d / W);
    const int q4 = W / 4;
    float s = 0.f;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int j0 = 0; j0 < nslab; ++j0) {
            const int j = rot ? (int)((j0 + t * 37) % nslab) : j0;
            for (int e = threadIdx.x; e < 32 * q4; e += blockDim.x) {
                const int r = e / q4, c = e % q4;
                const float4 v = __ldcs(reinterpret_cast<const float4*>(X + (t * 32 + r) * d + (int64_t)j * W) + c);
                s += v.x + v.y + v.z + v.w;
            }
        }
    }
    if (s == 12345.f) out[0] = s;
}

__device__ __forceinline__ float4 ldg_na(const float* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
// C4-style batches: 512 threads, each step = 16 float4 per thread issued together.
// mode 0: step = 32 consecutive rows x 1024 floats (rows of length d, first 1024 cols... contiguous when d == 1024)
// mode 1: step = 4 slabs x 32 rows x 256 floats (slab stride 256 floats, row stride d)
__global__ void __launch_bounds__(512, 1) batched(const float* __restrict__ X, int64_t n, int64_t d, int mode, float* out) {
    const int tid = threadIdx.x;
    float s = 0.f;
    const int64_t ntiles = n / 32;
    const int steps_per_tile = mode == 0 ? (int)(d / 1024) : (int)(d / 1024);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int st = 0; st < steps_per_tile; ++st) {
            float4 b[16];
            if (mode == 0) {
                const int c4 = tid % 256, r0 = tid / 256;   // 2 rows per iteration, 1024 floats per row
#pragma unroll
                for (int v = 0; v < 16; ++v) b[v] = ldg_na(X + (t * 32 + r0 + 2 * v) * d + st * 1024 + 4 * c4);
            } else {
                const int c4 = tid % 64, r0 = tid / 64;     // 8 rows per iteration, 256 floats per row
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        b[q * 4 + v] = ldg_na(X + (t * 32 + r0 + 8 * v) * d + (int64_t)(st * 4 + q) * 256 + 4 * c4);
            }
#pragma unroll
            for (int v = 0; v < 16; ++v) s += b[v].x + b[v].y + b[v].z + b[v].w;
        }
    }
    if (s == 12345.f) out[0] = s;
}

int main() {
    const int64_t n = 20000, d = 65536;
    float* X;
    cudaMalloc(&X, n * d * 4);
    cudaMemset(X, 0, n * d * 4);
    float* out;
    cudaMalloc(&out, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto report = [&](const char* name, auto launch) {
        launch();
        cudaEventRecord(a);
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 3;
        printf("%-40s %8.3f ms  %7.1f GB/s\n", name, ms, n * d * 4 / (ms * 1e-3) / 1e9);
    };
    report("contiguous float4 (148x1024 thr)", [&] { contiguous<<<148 * 4, 256>>>((const float4*)X, n * d / 4, out); });
    report("batched mode0 (32 rows x 4KB chunks)", [&] { batched<<<148, 512>>>(X, n, d, 0, out); });
    report("batched mode1 (4 slabs x 32 rows x 1KB)", [&] { batched<<<148, 512>>>(X, n, d, 1, out); });
    {
        // C4 shape: d = 1024 contiguous rows
        const int64_t n4 = n * d / 1024;
        report("batched mode0 d=1024 (fully contiguous)", [&] { batched<<<148, 512>>>(X, n4, 1024, 0, out); });
    }
    for (int W : {256, 1024, 4096, 16384}) {
        for (int rot : {0, 1}) {
            for (int blocks : {148, 296, 592}) {
                char name[128];
                snprintf(name, sizeof name, "slabs W=%d rot=%d grid=%d", W, rot, blocks);
                report(name, [&] { slabs<<<blocks, 512>>>(X, n, d, W, rot, out); });
            }
        }
    }
    return 0;
}
