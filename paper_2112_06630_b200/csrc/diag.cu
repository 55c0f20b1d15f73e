// Diagnostics library (libknng_diag.so): measured FP32 FFMA peak of the
// device, the denominator of the local join's FP32 roofline (MEASURED_PEAKS.json
// records only HBM and bf16 tensor peaks).  Not on the hot path.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

// 16 independent FFMA chains per thread, 3-register form (the form the join
// issues), so the measurement reflects the fma pipe at full occupancy.
__global__ void __launch_bounds__(256) ffma_kernel(float* out, int iters, float a, float b) {
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = float(threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 12345.678f) out[0] = s;  // keep the chains live
}

// Packed FP32x2 (FFMA2) chains, all operands in registers.
__global__ void __launch_bounds__(256) ffma2_kernel(float* out, int iters, float a, float b) {
    float2 x[8];
    const float2 va = make_float2(a, a * 0.5f), vb = make_float2(b, b * 2.0f);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = make_float2(float(threadIdx.x + i), float(i));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(x[i], va, vb);
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
    if (s == 12345.678f) out[0] = s;
}

// Legacy integer MMA (mma.sync m16n8k32 u8 x u8 -> s32, the byte-valued
// join's instruction), 8 independent accumulator chains per warp.
__global__ void __launch_bounds__(512) imma_kernel(int* out, int iters) {
    int acc[8][4];
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[c][r] = 0;
    const uint32_t a0 = threadIdx.x * 0x01010101u, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    const uint32_t b0 = a0 ^ 0x5a5a5a5au, b1 = a0 ^ 0x3c3c3c3cu;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
            asm volatile(
                "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
                "{%8,%9}, {%0,%1,%2,%3};\n"
                : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    int s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
    if (s == 123456789) out[0] = s;
}

}  // namespace

// Integer tensor-core peak of the legacy MMA path (TOPS, 2 ops per MAC).
extern "C" int knng_diag_imma_peak(int device, double* tops) {
    if (cudaSetDevice(device) != cudaSuccess) return 2;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    int* out = nullptr;
    if (cudaMalloc(&out, sizeof(int)) != cudaSuccess) return 2;
    const int blocks = sms, threads = 512, iters = 1 << 12;
    for (int w = 0; w < 3; ++w) imma_kernel<<<blocks, threads>>>(out, iters);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) imma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double macs = 16.0 * 8 * 32 * 8 * double(iters) * (threads / 32) * blocks * reps;
    *tops = 2.0 * macs / (double(ms) * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

// FP32 peak as the max of the scalar-FFMA and packed-FFMA2 measurements.
extern "C" int knng_diag_ffma2_peak(int device, double* tflops) {
    if (cudaSetDevice(device) != cudaSuccess) return 2;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float* out = nullptr;
    if (cudaMalloc(&out, sizeof(float)) != cudaSuccess) return 2;
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    for (int w = 0; w < 5; ++w) ffma2_kernel<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) ffma2_kernel<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    *tflops = 2.0 * 16.0 * double(iters) * double(blocks) * threads * reps / (double(ms) * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

extern "C" int knng_diag_ffma_peak(int device, double* tflops, double* ms_out) {
    if (cudaSetDevice(device) != cudaSuccess) return 2;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float* out = nullptr;
    if (cudaMalloc(&out, sizeof(float)) != cudaSuccess) return 2;
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    // warm up (clocks ramp)
    for (int w = 0; w < 5; ++w) ffma_kernel<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) ffma_kernel<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 16.0 * double(iters) * double(blocks) * threads * reps;
    *tflops = flops / (double(ms) * 1e-3) / 1e12;
    if (ms_out) *ms_out = ms / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
