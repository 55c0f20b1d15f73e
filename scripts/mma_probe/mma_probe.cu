// Latency / throughput of legacy mma.sync m16n8k8 TF32 on this GPU
// (diagnostic for the screened join, csrc/join_tc.cu).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int CH>
__global__ void probe(float* out, int iters) {
    float acc[CH][4];
    for (int c = 0; c < CH; ++c) for (int r = 0; r < 4; ++r) acc[c][r] = 0.f;
    uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile(
                "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
                "{%8,%9}, {%0,%1,%2,%3};\n"
                : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int c = 0; c < CH; ++c) for (int r = 0; r < 4; ++r) s += acc[c][r];
    if (s == 1.2345f) out[0] = s;
}

template <int CH>
void run(int warps, float* out) {
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    probe<CH><<<148, warps * 32>>>(out, iters);
    cudaEventRecord(e0);
    probe<CH><<<148, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double cyc = ms * 1e-3 * 1.965e9;
    const double mmas_per_sm = double(iters) * CH * warps;
    printf("warps/SM %2d chains %d: %.1f cycles per dependent mma per warp, %.2f mma/cycle/SM, %.0f TFLOP/s tf32\n",
           warps, CH, cyc / iters / CH * CH, mmas_per_sm / cyc,
           mmas_per_sm * 148 * 2 * 16 * 8 * 8 / (ms * 1e-3) / 1e12);
}

int main() {
    float* out; cudaMalloc(&out, 4);
    run<1>(1, out); run<1>(4, out); run<4>(4, out); run<8>(4, out); run<8>(8, out); run<8>(16, out);
    run<4>(16, out); run<8>(32, out);
    return 0;
}
