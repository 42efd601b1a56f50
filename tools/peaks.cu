// tools/peaks.cu -- measured denominators for the roofline of the GRCA path ("Measure an FP32
// FMA microbenchmark and an L2 u64 atomicMin microbenchmark on the box, and use those as the denominators").
//   ffma   : FP32 FFMA lane-instructions / s  (8 independent chains per thread, full occupancy)
//   ffma2  : packed FFMA2 (fp32x2) lane-instructions / s (each does 2 FMAs per lane)
//   red    : u64 RED.MIN (atomicMin, result unused) / s into a 33.5 MB buffer (the C4 hit-key buffer size,
//            L2-resident), random addresses (one sector per op) and lane-consecutive addresses
// Host entry: peaks_run(kind, &value, &ms) -> 0 on success.  Measurement harness, not part of libgrca.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void k_ffma(float *out, int iters) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3f + k;
    const float b = 0.99999f, c = 1e-7f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = __fmaf_rn(a[k], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 123456.789f) out[blockIdx.x] = s;
}

__global__ void k_ffma2(float *out, int iters) {
    float2 a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = make_float2(threadIdx.x * 1e-3f + k, k * 0.5f);
    const float2 b = make_float2(0.99999f, 0.99998f), c = make_float2(1e-7f, 2e-7f);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = __ffma2_rn(a[k], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k].x + a[k].y;
    if (s == 123456.789f) out[blockIdx.x] = s;
}

__global__ void k_red(unsigned long long *buf, unsigned mask, int iters, int coalesced) {
    const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned x = tid * 2654435761u + 12345u;
    for (int i = 0; i < iters; ++i) {
        x = x * 1664525u + 1013904223u;
        const unsigned a = coalesced ? ((tid + (unsigned)i * gridDim.x * blockDim.x) & mask) : (x & mask);
        atomicMin(buf + a, ((unsigned long long)(x >> 8) << 32) | x);   // result unused -> RED.MIN
    }
}

extern "C" int peaks_run(int kind, double *value, double *ms_out) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int block = 256, grid = sms * 8;
    float *out = nullptr;
    unsigned long long *buf = nullptr;
    const unsigned nbuf = 1u << 22;   // 4,194,304 keys = 33.5 MB
    if (cudaMalloc(&out, sizeof(float) * grid) != cudaSuccess) return 2;
    if (kind >= 2 && cudaMalloc(&buf, sizeof(unsigned long long) * nbuf) != cudaSuccess) return 2;
    if (buf) cudaMemset(buf, 0xff, sizeof(unsigned long long) * nbuf);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = kind < 2 ? 4096 : 256;
    auto launch = [&]() {
        if (kind == 0) k_ffma<<<grid, block>>>(out, iters);
        else if (kind == 1) k_ffma2<<<grid, block>>>(out, iters);
        else k_red<<<grid, block>>>(buf, nbuf - 1, iters, kind == 3);
    };
    launch();   // warm-up (clocks, L2)
    launch();
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double threads = (double)grid * block;
    const double per_thread = kind < 2 ? (double)iters * 32.0 : (double)iters;   // instructions or REDs
    *value = threads * per_thread * reps / (ms * 1e-3);
    *ms_out = ms / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    cudaFree(buf);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
