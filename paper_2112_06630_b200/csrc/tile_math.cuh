// Exact lane-split tile arithmetic shared by the FP32 join kernels (join.cu,
// join_gl.cu).  Compile the including file with --fmad=false: the unfused
// path must stay a rounded square followed by an add.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace knng_cuda {

// Offset of candidate r's row in its node's proposal block (nn new, m = nn + no
// candidates): word 0 = count, then up to m - 1 (new r) or nn (old r) keys
// (distance bits << 32 | partner id).
__device__ __forceinline__ size_t prow(uint32_t r, uint32_t nn, uint32_t m) {
    return r < nn ? size_t(r) * m : size_t(nn) * m + size_t(r - nn) * (nn + 1);
}

__device__ __forceinline__ float acc_at(const float2 (&acc)[32], uint32_t p) {
    return (p & 1u) ? acc[p >> 1].y : acc[p >> 1].x;
}

// Reduce-scatter of the 64 per-lane partial sums over a group's 8 lanes in
// the reference's tree order ((0+1)+(2+3))+((4+5)+(6+7)) (distance.hpp:29-51);
// lane l8 = b0 + 2 b1 + 4 b2 ends with the 8 sums of accumulator row
// X = 4 b0 + 2 b1 + b2 (floats 8X .. 8X + 7 of acc).
__device__ __forceinline__ void group_reduce64(const float2 (&acc)[32], uint32_t l8,
                                               float (&row)[8]) {
    const bool b0 = l8 & 1u, b1 = (l8 >> 1) & 1u, b2 = (l8 >> 2) & 1u;
    float r32[32];
#pragma unroll
    for (uint32_t j = 0; j < 32; ++j) {
        const float send = b0 ? acc_at(acc, j) : acc_at(acc, 32 + j);
        const float keep = b0 ? acc_at(acc, 32 + j) : acc_at(acc, j);
        r32[j] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 1));
    }
    float r16[16];
#pragma unroll
    for (uint32_t j = 0; j < 16; ++j) {
        const float send = b1 ? r32[j] : r32[16 + j];
        const float keep = b1 ? r32[16 + j] : r32[j];
        r16[j] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 2));
    }
#pragma unroll
    for (uint32_t j = 0; j < 8; ++j) {
        const float send = b2 ? r16[j] : r16[8 + j];
        const float keep = b2 ? r16[8 + j] : r16[j];
        row[j] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 4));
    }
}

// The accumulator row a lane holds after group_reduce64.
__device__ __forceinline__ uint32_t reduced_row(uint32_t l8) {
    return 4u * (l8 & 1u) + 2u * ((l8 >> 1) & 1u) + ((l8 >> 2) & 1u);
}

}  // namespace knng_cuda
