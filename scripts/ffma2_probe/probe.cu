// What FFMA2 rate can the join's instruction pattern reach at the join's
// occupancy (128-thread CTAs, 4 per SM, ~120 registers)?  Each thread keeps 25
// float2 accumulators and per step does the 5 x 10 tile's segment:
//   diff = fma2(b[j], -1, a[x]);  acc[5x + j] = fma2(diff, diff, acc[5x + j])
// with the 15 operands (a) held in registers, (b) reloaded from shared memory
// every step as the join does (conflict-free addresses), (c) as (b) with the
// join's row pitch and four groups per warp reading four different rows.
// Prints FFMA2 per clock per SM sub-partition (peak 0.5) for each variant.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kPitch = 36;

template <int kMode>
__global__ void __launch_bounds__(128, 4) pattern(float* out, const float* in, int steps, float seed) {
    extern __shared__ float smem[];
    const int tid = threadIdx.x, l8 = tid & 7, group = tid >> 3;
    for (int i = tid; i < 112 * kPitch; i += 128) smem[i] = in[i % 1024] + seed;
    __syncthreads();
    float2 acc[25];
#pragma unroll
    for (int p = 0; p < 25; ++p) acc[p] = make_float2(0.f, 0.f);
    float a[5];
    float2 b[5];
#pragma unroll
    for (int x = 0; x < 5; ++x) {
        a[x] = seed * (x + 1) + tid;
        b[x] = make_float2(seed * x, seed + x + tid);
    }
    const float2 m1 = make_float2(-1.f, -1.f);
    // mode 1: every thread its own 15 consecutive words; mode 2: the join's layout
    const float* pa = kMode == 2 ? smem + (group * 5 % 100) * kPitch + l8 : smem + tid;
    const float* pb = kMode == 2 ? smem + ((group * 10 + 5) % 100) * kPitch + l8 : smem + 128 * 5 + tid;
    for (int s = 0; s < steps; ++s) {
        if (kMode >= 1) {
            const int o = (s & 3) * 8;
            if (kMode == 2) {
#pragma unroll
                for (int x = 0; x < 5; ++x) a[x] = pa[x * kPitch + o];
#pragma unroll
                for (int j = 0; j < 5; ++j)
                    b[j] = make_float2(pb[(2 * j) * kPitch + o], pb[(2 * j + 1) * kPitch + o]);
            } else {
#pragma unroll
                for (int x = 0; x < 5; ++x) a[x] = pa[x * 128 + (s & 3) * 1024];
#pragma unroll
                for (int j = 0; j < 5; ++j)
                    b[j] = make_float2(pb[(2 * j) * 128 + (s & 3) * 1024], pb[(2 * j + 1) * 128 + (s & 3) * 1024]);
            }
        } else {
#pragma unroll
            for (int x = 0; x < 5; ++x) a[x] += 1.0f;  // keep diff from being hoisted
        }
#pragma unroll
        for (int x = 0; x < 5; ++x) {
            const float2 ax = make_float2(a[x], a[x]);
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                const float2 d = __ffma2_rn(b[j], m1, ax);
                acc[5 * x + j] = __ffma2_rn(d, d, acc[5 * x + j]);
            }
        }
    }
    float sum = 0.f;
#pragma unroll
    for (int p = 0; p < 25; ++p) sum += acc[p].x + acc[p].y;
    if (sum == 12345.678f) out[0] = sum;
}

template <int kMode>
void run(const char* name, float* out, const float* in, int sms, double clock_ghz) {
    const int steps = 1 << 14, blocks = sms * 4, smem = 112 * kPitch * 4 * 3;
    cudaFuncSetAttribute(pattern<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int w = 0; w < 3; ++w) pattern<kMode><<<blocks, 128, smem>>>(out, in, steps, 0.5f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) pattern<kMode><<<blocks, 128, smem>>>(out, in, steps, 0.5f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    // warp-level FFMA2 per SM sub-partition: 4 warps per CTA, 4 CTAs per SM = 4 warps per sub-partition
    const double ffma2_per_smsp = 50.0 * steps * 4 * reps;
    const double clocks = double(ms) * 1e-3 * clock_ghz * 1e9;
    printf("{\"variant\": \"%s\", \"ms\": %.3f, \"ffma2_per_clk_per_smsp\": %.4f, \"frac_of_peak\": %.4f, \"err\": \"%s\"}\n",
           name, ms / reps, ffma2_per_smsp / clocks, ffma2_per_smsp / clocks / 0.5,
           cudaGetErrorString(cudaGetLastError()));
}


// (d) as (c), four segments per loop trip with the next segment's 15 loads
// issued before the current segment's arithmetic (explicit double buffer).
// (e) one thread = two reference lanes of ONE pair per float2: a 5 x 5 tile per
// 4-thread group, operands by 8-byte loads (10 LDS.64 per 50 FFMA2).
template <int kMode>
__global__ void __launch_bounds__(128, 4) pattern2(float* out, const float* in, int steps, float seed) {
    extern __shared__ float smem[];
    const int tid = threadIdx.x, l8 = tid & 7, group = tid >> 3;
    for (int i = tid; i < 112 * kPitch; i += 128) smem[i] = in[i % 1024] + seed;
    __syncthreads();
    float2 acc[25];
#pragma unroll
    for (int p = 0; p < 25; ++p) acc[p] = make_float2(0.f, 0.f);
    const float2 m1 = make_float2(-1.f, -1.f);
    if (kMode == 3) {
        const float* pa = smem + (group * 5 % 100) * kPitch + l8;
        const float* pb = smem + ((group * 10 + 5) % 100) * kPitch + l8;
        float a0[5], a1[5];
        float2 b0[5], b1[5];
#define LOAD(A, B, o)                                                                          \
    _Pragma("unroll") for (int x = 0; x < 5; ++x) A[x] = pa[x * kPitch + (o)];                 \
    _Pragma("unroll") for (int j = 0; j < 5; ++j)                                              \
        B[j] = make_float2(pb[(2 * j) * kPitch + (o)], pb[(2 * j + 1) * kPitch + (o)]);
#define MATH(A, B)                                                                             \
    _Pragma("unroll") for (int x = 0; x < 5; ++x) {                                            \
        const float2 ax = make_float2(A[x], A[x]);                                             \
        _Pragma("unroll") for (int j = 0; j < 5; ++j) {                                        \
            const float2 d = __ffma2_rn(B[j], m1, ax);                                         \
            acc[5 * x + j] = __ffma2_rn(d, d, acc[5 * x + j]);                                 \
        }                                                                                      \
    }
        LOAD(a0, b0, 0)
        for (int s = 0; s < steps; s += 4) {
            const int w = s & 4;  // keeps the loads inside the loop
            LOAD(a1, b1, 8 + w)
            MATH(a0, b0)
            LOAD(a0, b0, 16 + w)
            MATH(a1, b1)
            LOAD(a1, b1, 24 + w)
            MATH(a0, b0)
            LOAD(a0, b0, 4 - w)
            MATH(a1, b1)
        }
    } else {
        // 4-thread groups: thread q of a group holds reference lanes 2q, 2q + 1
        const int q = tid & 3, g4 = tid >> 2;
        const float2* pa = reinterpret_cast<const float2*>(smem + (g4 * 5 % 100) * kPitch) + q;
        const float2* pb = reinterpret_cast<const float2*>(smem + ((g4 * 5 + 50) % 100) * kPitch) + q;
        for (int s = 0; s < steps; ++s) {
            const int o = (s & 3) * 4;  // float2 units: 8 floats per segment
            float2 a[5], b[5];
#pragma unroll
            for (int x = 0; x < 5; ++x) a[x] = pa[x * (kPitch / 2) + o];
#pragma unroll
            for (int j = 0; j < 5; ++j) b[j] = pb[j * (kPitch / 2) + o];
#pragma unroll
            for (int x = 0; x < 5; ++x)
#pragma unroll
                for (int j = 0; j < 5; ++j) {
                    const float2 d = __ffma2_rn(b[j], m1, a[x]);
                    acc[5 * x + j] = __ffma2_rn(d, d, acc[5 * x + j]);
                }
        }
    }
    float sum = 0.f;
#pragma unroll
    for (int p = 0; p < 25; ++p) sum += acc[p].x + acc[p].y;
    if (sum == 12345.678f) out[0] = sum;
}

template <int kMode>
void run2(const char* name, float* out, const float* in, int sms, double clock_ghz, int ctas = 4) {
    const int steps = 1 << 14, blocks = sms * ctas, smem = ctas == 4 ? 112 * kPitch * 4 * 3 : 220 * 1024 / ctas;
    cudaFuncSetAttribute(pattern2<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int w = 0; w < 3; ++w) pattern2<kMode><<<blocks, 128, smem>>>(out, in, steps, 0.5f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) pattern2<kMode><<<blocks, 128, smem>>>(out, in, steps, 0.5f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ffma2_per_smsp = 50.0 * steps * ctas * reps;
    const double clocks = double(ms) * 1e-3 * clock_ghz * 1e9;
    printf("{\"variant\": \"%s\", \"ctas_per_sm\": %d, \"ms\": %.3f, \"ffma2_per_clk_per_smsp\": %.4f, \"frac_of_peak\": %.4f, \"err\": \"%s\"}\n",
           name, ctas, ms / reps, ffma2_per_smsp / clocks, ffma2_per_smsp / clocks / 0.5,
           cudaGetErrorString(cudaGetLastError()));
}

// (f) two 5 x 10 tiles per thread (two accumulator sets, ~200 registers), 2 CTAs
// per SM: what a pass of 32 tiles on 16 groups could reach -- a whole
// iteration-1 node per pass at half the passes.
__global__ void __launch_bounds__(128, 2) pattern_two(float* out, const float* in, int steps, float seed) {
    extern __shared__ float smem[];
    const int tid = threadIdx.x, l8 = tid & 7, group = tid >> 3;
    for (int i = tid; i < 112 * kPitch; i += 128) smem[i] = in[i % 1024] + seed;
    __syncthreads();
    float2 acc0[25], acc1[25];
#pragma unroll
    for (int p = 0; p < 25; ++p) acc0[p] = acc1[p] = make_float2(0.f, 0.f);
    const float2 m1 = make_float2(-1.f, -1.f);
    const float* pa0 = smem + (group * 5 % 100) * kPitch + l8;
    const float* pb0 = smem + ((group * 10 + 5) % 100) * kPitch + l8;
    const float* pa1 = smem + ((group * 5 + 40) % 100) * kPitch + l8;
    const float* pb1 = smem + ((group * 10 + 55) % 100) * kPitch + l8;
    for (int s = 0; s < steps; ++s) {
        const int o = (s & 3) * 8;
        float a0[5], a1[5];
        float2 b0[5], b1[5];
#pragma unroll
        for (int x = 0; x < 5; ++x) {
            a0[x] = pa0[x * kPitch + o];
            a1[x] = pa1[x * kPitch + o];
        }
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            b0[j] = make_float2(pb0[(2 * j) * kPitch + o], pb0[(2 * j + 1) * kPitch + o]);
            b1[j] = make_float2(pb1[(2 * j) * kPitch + o], pb1[(2 * j + 1) * kPitch + o]);
        }
#pragma unroll
        for (int x = 0; x < 5; ++x) {
            const float2 ax0 = make_float2(a0[x], a0[x]), ax1 = make_float2(a1[x], a1[x]);
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                const float2 d0 = __ffma2_rn(b0[j], m1, ax0);
                acc0[5 * x + j] = __ffma2_rn(d0, d0, acc0[5 * x + j]);
                const float2 d1 = __ffma2_rn(b1[j], m1, ax1);
                acc1[5 * x + j] = __ffma2_rn(d1, d1, acc1[5 * x + j]);
            }
        }
    }
    float sum = 0.f;
#pragma unroll
    for (int p = 0; p < 25; ++p) sum += acc0[p].x + acc0[p].y + acc1[p].x + acc1[p].y;
    if (sum == 12345.678f) out[0] = sum;
}

void run_two(float* out, const float* in, int sms, double clock_ghz) {
    const int steps = 1 << 13, ctas = 2, blocks = sms * ctas, smem = 100 * 1024;
    cudaFuncSetAttribute(pattern_two, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int w = 0; w < 3; ++w) pattern_two<<<blocks, 128, smem>>>(out, in, steps, 0.5f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) pattern_two<<<blocks, 128, smem>>>(out, in, steps, 0.5f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ffma2_per_smsp = 100.0 * steps * ctas * reps;
    const double clocks = double(ms) * 1e-3 * clock_ghz * 1e9;
    printf("{\"variant\": \"two 5 x 10 tiles per thread, load both then compute both\", \"ctas_per_sm\": %d, \"ms\": %.3f, \"ffma2_per_clk_per_smsp\": %.4f, \"frac_of_peak\": %.4f, \"err\": \"%s\"}\n",
           ctas, ms / reps, ffma2_per_smsp / clocks, ffma2_per_smsp / clocks / 0.5,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms = 0, khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double ghz = 1.965;  // SM clock under load on this pool's B200s (bench `clocks`)
    float *out, *in;
    cudaMalloc(&out, 4);
    cudaMalloc(&in, 4096);
    cudaMemset(in, 0, 4096);
    printf("{\"sms\": %d, \"max_clock_khz\": %d, \"assumed_ghz\": %.3f}\n", sms, khz, ghz);
    run<0>("operands in registers", out, in, sms, ghz);
    run<1>("15 shared loads per 50 FFMA2, conflict-free", out, in, sms, ghz);
    run<2>("15 shared loads per 50 FFMA2, join layout (pitch 36, 4 groups per warp)", out, in, sms, ghz);
    run2<3>("join layout, next segment loaded before this segment's arithmetic", out, in, sms, ghz);
    run2<3>("join layout, next segment loaded before this segment's arithmetic", out, in, sms, ghz, 3);
    run2<3>("join layout, next segment loaded before this segment's arithmetic", out, in, sms, ghz, 2);
    run2<4>("5 x 5 tile per 4-thread group, 10 LDS.64 per 50 FFMA2", out, in, sms, ghz);
    run_two(out, in, sms, ghz);
    return 0;
}
