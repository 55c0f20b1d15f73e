// Local join (compute_step, reference descent.hpp:82-153) for byte-valued
// data on the integer tensor cores, bit-identical to the reference.
//
// When every coordinate is an integer in [0, 255] (pixel intensities,
// SIFT-style descriptors — BASELINE config C2), every term (a_j - b_j)^2 is an
// integer below 2^16 and each of the reference's eight strided lane sums
// (lane l = elements 8c + l, distance.hpp:35-88) is an integer below 2^24
// whenever stride / 8 <= 258.  Every FP32 partial sum of a lane is then exact,
// whichever of the reference's paths (FMA-contracted tiles or unfused scalar)
// forms it, so
//     lane_l(a, b) = |a|_l^2 + |b|_l^2 - 2 <a, b>_l          (exact integers)
// and the reference's distance is the FP32 tree ((0+1)+(2+3))+((4+5)+(6+7))
// of those lane sums.  This kernel forms the eight per-lane dot products with
// mma.sync m16n8k32 u8 x u8 -> s32 on a lane-major byte copy of the data
// (8 x Kl bytes per row, Kl = stride / 8 rounded up to 32), adds the per-lane
// squared norms, and applies the tree with __fadd_rn — every distance
// bit-identical to the reference (tests/test_gpu_parity.py runs C2 through
// this path; tests/test_gpu_u8.py compares it with the FP32 tile kernel).
//
// One warp per active node (no shared staging: the byte copy, n x 8 Kl bytes,
// is 70 MB for C2 and stays in L2); per (16-row block of new candidates,
// 4 column blocks) the warp runs 8 lanes x Kl / 32 MMAs and writes the
// proposals that beat an endpoint's row maximum into the node's proposal
// block in join.cu's format.
#include <cstdio>

#include "kernels.cuh"

namespace knng_cuda {

namespace {

constexpr uint32_t kUWarps = 8;                 // warps per CTA, one node each
constexpr uint32_t kUMaxM = 2 * kMaxCap;

struct U8Warp {
    uint32_t rid[kUMaxM];     // combined index -> data row
    float rmx[kUMaxM];        // prefilter bound (row maximum), +inf when unfiltered
    uint32_t rowcnt[kUMaxM];  // proposals kept per candidate row
};

__device__ __forceinline__ void mma_u8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                       uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ size_t u8_prow(uint32_t r, uint32_t nn, uint32_t m) {
    return r < nn ? size_t(r) * m : size_t(nn) * m + size_t(r - nn) * (nn + 1);
}

// Byte-layout of one row: lane l occupies bytes [l Kl, (l + 1) Kl); inside a
// lane, each 32-byte k-chunk is permuted so that MMA thread t's eight bytes
// (k = 4t..4t+3 and 16+4t..16+4t+3 of the chunk) are contiguous at 8t: one
// 8-byte load per fragment pair.  The permutation is the same for both MMA
// operands, and integer dot products do not depend on the order of terms.
__device__ __forceinline__ uint32_t u8_pos(uint32_t kk) {  // kk in [0, 32)
    const uint32_t t = (kk & 15u) >> 2, h = kk >> 4, b = kk & 3u;
    return 8 * t + 4 * h + b;
}

// All coordinates integral in [0, 255]?  flag starts at 1; any miss clears it.
__global__ void u8_check_kernel(const float* __restrict__ data, size_t count, uint32_t* flag) {
    bool ok = true;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += size_t(gridDim.x) * blockDim.x) {
        const float x = data[i];
        ok &= x >= 0.0f && x <= 255.0f && x == rintf(x);
    }
    if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31u) == 0) atomicAnd(flag, 0u);
}

// Lane-major byte copy and per-lane squared norms (exact integers).  One warp
// per row; lane l of the warp owns reference lane l % 8 ... every thread
// handles whole 32-byte k-chunks of one lane.
__global__ void u8_pack_kernel(const float* __restrict__ data, uint32_t n, uint32_t stride,
                               uint32_t kl, uint8_t* __restrict__ packed,
                               int32_t* __restrict__ lnorm) {
    const uint32_t row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31u;
    if (row >= n) return;
    const float* x = data + size_t(row) * stride;
    uint8_t* out = packed + size_t(row) * 8 * kl;
    const uint32_t chunks = kl / 32;  // k-chunks per lane
    int32_t nrm = 0;                  // lane (lane & 7)'s partial norm
    for (uint32_t w = lane; w < 8 * chunks; w += 32) {
        const uint32_t l = w % 8, ch = w / 8;
        uint8_t buf[32];
#pragma unroll
        for (uint32_t kk = 0; kk < 32; ++kk) {
            const uint32_t c = ch * 32 + kk, e = 8 * c + l;
            const uint32_t v = e < stride ? uint32_t(x[e]) : 0u;
            buf[u8_pos(kk)] = uint8_t(v);
            nrm += int32_t(v * v);
        }
        uint4* dst = reinterpret_cast<uint4*>(out + l * kl + ch * 32);
        dst[0] = *reinterpret_cast<const uint4*>(buf);
        dst[1] = *reinterpret_cast<const uint4*>(buf + 16);
    }
    // lanes congruent mod 8 hold the same reference lane
    nrm += __shfl_xor_sync(0xffffffffu, nrm, 8);
    nrm += __shfl_xor_sync(0xffffffffu, nrm, 16);
    if (lane < 8) lnorm[size_t(row) * 8 + lane] = nrm;
}

__global__ void __launch_bounds__(kUWarps * 32, 2) join_u8_kernel(GraphView g, CandView c,
                                                               IterCounters* ctr,
                                                               const uint8_t* __restrict__ packed,
                                                               const int32_t* __restrict__ lnorm,
                                                               uint32_t kl) {
    __shared__ U8Warp shw[kUWarps];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t gq = lane >> 2, t = lane & 3u;
    U8Warp& W = shw[warp];
    if (ctr->overflow) return;
    const uint32_t n_active = ctr->active, cap = c.cap;
    const size_t row_bytes = size_t(8) * kl;
    const uint32_t chunks = kl / 32;
    for (;;) {
        uint32_t a = 0;
        if (lane == 0) a = atomicAdd(&ctr->work, 1u);
        a = __shfl_sync(0xffffffffu, a, 0);
        if (a >= n_active) break;
        const uint4 rec = c.arec[a];
        const uint32_t u = rec.x, nn = rec.y & 0xffffu, no = rec.y >> 16, m = nn + no;
        uint64_t* const D = c.D + (uint64_t(rec.z) | (uint64_t(rec.w) << 32));
        for (uint32_t x = lane; x < m; x += 32) {
            const size_t pos = size_t(u) * 2 * cap + (x < nn ? x : cap + x - nn);
            W.rid[x] = c.ids[pos];
            W.rmx[x] = c.filter ? c.cmax[pos] : __int_as_float(0x7f800000);
            W.rowcnt[x] = 0;
        }
        __syncwarp();
        // padding rows of the last 16 / 8 blocks: any valid row (read, unused)
        for (uint32_t x = m + lane; x < kUMaxM; x += 32) W.rid[x] = W.rid[0];
        __syncwarp();
        const uint32_t nmi = (nn + 15) / 16, nnj = (m + 7) / 8;
        for (uint32_t mi = 0; mi < nmi; ++mi) {
            const uint8_t* pa0 = packed + size_t(W.rid[16 * mi + gq]) * row_bytes + 8 * t;
            const uint8_t* pa1 = packed + size_t(W.rid[16 * mi + gq + 8]) * row_bytes + 8 * t;
            const int32_t* na0 = lnorm + size_t(W.rid[16 * mi + gq]) * 8;
            const int32_t* na1 = lnorm + size_t(W.rid[16 * mi + gq + 8]) * 8;
            // column blocks whose pairs all lie on or below the diagonal of
            // the new x new triangle are skipped
            for (uint32_t njb = 2 * mi; njb < nnj; njb += 4) {
                const uint8_t* pb[4];
                const int32_t* nb0[4];
                const int32_t* nb1[4];
#pragma unroll
                for (uint32_t q = 0; q < 4; ++q) {
                    const uint32_t col = min(8 * (njb + q) + gq, kUMaxM - 1);
                    const uint32_t cn = min(8 * (njb + q) + 2 * t, kUMaxM - 2);
                    pb[q] = packed + size_t(W.rid[col]) * row_bytes + 8 * t;
                    nb0[q] = lnorm + size_t(W.rid[cn]) * 8;
                    nb1[q] = lnorm + size_t(W.rid[cn + 1]) * 8;
                }
                // tree partials of the 4 x 4 C elements: s01/s45 after odd
                // lanes, s0123 after lane 3
                float part[4][4][3];
#pragma unroll
                for (uint32_t l = 0; l < 8; ++l) {
                    int acc[4][4];
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q)
#pragma unroll
                        for (uint32_t r = 0; r < 4; ++r) acc[q][r] = 0;
                    for (uint32_t ch = 0; ch < chunks; ++ch) {
                        const size_t o = size_t(l) * kl + 32 * ch;
                        const uint2 A0 = __ldg(reinterpret_cast<const uint2*>(pa0 + o));
                        const uint2 A1 = __ldg(reinterpret_cast<const uint2*>(pa1 + o));
#pragma unroll
                        for (uint32_t q = 0; q < 4; ++q) {
                            if (njb + q < nnj) {
                                const uint2 B = __ldg(reinterpret_cast<const uint2*>(pb[q] + o));
                                mma_u8(acc[q], A0.x, A1.x, A0.y, A1.y, B.x, B.y);
                            }
                        }
                    }
                    // lane sums (exact integers < 2^24) into the tree
                    const int32_t a_n0 = __ldg(na0 + l), a_n1 = __ldg(na1 + l);
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q) {
                        if (njb + q >= nnj) continue;
                        const int32_t b_n0 = __ldg(nb0[q] + l);  // column 2t
                        const int32_t b_n1 = __ldg(nb1[q] + l);  // column 2t + 1
#pragma unroll
                        for (uint32_t r = 0; r < 4; ++r) {
                            const int32_t an = r < 2 ? a_n0 : a_n1;
                            const int32_t bn = (r & 1u) ? b_n1 : b_n0;
                            const float s = float(an + bn - 2 * acc[q][r]);
                            float* p = part[q][r];
                            if (l == 0 || l == 2 || l == 4 || l == 6) {
                                p[l == 2 || l == 6 ? 1 : 0] = s;
                            } else if (l == 1 || l == 5) {
                                p[0] = __fadd_rn(p[0], s);  // (0+1) / (4+5)
                            } else if (l == 3) {
                                p[2] = __fadd_rn(p[0], __fadd_rn(p[1], s));  // (0+1)+(2+3)
                            } else {  // l == 7
                                p[0] = __fadd_rn(p[2], __fadd_rn(p[0], __fadd_rn(p[1], s)));
                            }
                        }
                    }
                }
                // proposals of the 4 x 4 C elements
#pragma unroll
                for (uint32_t q = 0; q < 4; ++q) {
                    if (njb + q >= nnj) continue;
#pragma unroll
                    for (uint32_t r = 0; r < 4; ++r) {
                        const uint32_t i = 16 * mi + gq + 8 * (r >> 1);
                        const uint32_t j = 8 * (njb + q) + 2 * t + (r & 1u);
                        if (i >= nn || j >= m || (j < nn && j <= i)) continue;
                        const uint32_t id_i = W.rid[i], id_j = W.rid[j];
                        // an id listed twice pairs with itself: try_insert
                        // ignores self (graph.hpp:116-129)
                        if (c.filter && id_i == id_j) continue;
                        const float dist = part[q][r][0];
                        if (dist < W.rmx[i]) {
                            const uint32_t pos = atomicAdd(&W.rowcnt[i], 1u);
                            D[u8_prow(i, nn, m) + 1 + pos] = pack_key(dist, id_j);
                        }
                        if (dist < W.rmx[j]) {
                            const uint32_t pos = atomicAdd(&W.rowcnt[j], 1u);
                            D[u8_prow(j, nn, m) + 1 + pos] = pack_key(dist, id_i);
                        }
                    }
                }
            }
        }
        __syncwarp();
        for (uint32_t x = lane; x < m; x += 32) D[u8_prow(x, nn, m)] = W.rowcnt[x];
        __syncwarp();
    }
}

uint32_t u8_sm_count() {
    static uint32_t v = 0;
    if (!v) {
        int dev = 0, x = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&x, cudaDevAttrMultiProcessorCount, dev);
        v = x > 0 ? uint32_t(x) : 148u;
    }
    return v;
}

}  // namespace

uint32_t u8_lane_bytes(uint32_t stride) { return (stride / 8 + 31) / 32 * 32; }

bool u8_eligible(const float* data, uint32_t n, uint32_t stride, uint32_t* d_flag,
                 cudaStream_t s) {
    // lane sums stay below 2^24: (stride / 8) * 255^2 < 2^24
    if (stride / 8 > 258) return false;
    const uint32_t one = 1;
    cudaMemcpyAsync(d_flag, &one, sizeof(uint32_t), cudaMemcpyHostToDevice, s);
    u8_check_kernel<<<4 * u8_sm_count(), 256, 0, s>>>(data, size_t(n) * stride, d_flag);
    uint32_t h = 0;
    cudaMemcpyAsync(&h, d_flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    return h == 1;
}

void launch_u8_pack(const float* data, uint32_t n, uint32_t stride, uint8_t* packed,
                    int32_t* lnorm, cudaStream_t s) {
    u8_pack_kernel<<<uint32_t((size_t(n) * 32 + 255) / 256), 256, 0, s>>>(
        data, n, stride, u8_lane_bytes(stride), packed, lnorm);
}

void launch_join_u8(const GraphView& g, const CandView& c, IterCounters* ctr, uint32_t max_active,
                    const uint8_t* packed, const int32_t* lnorm, cudaStream_t s) {
    if (!max_active) return;
    static int per_sm = 0;
    if (!per_sm) {
        int v = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, join_u8_kernel, int(kUWarps * 32), 0);
        per_sm = v < 1 ? 1 : v;
    }
    uint32_t grid = u8_sm_count() * uint32_t(per_sm);
    const uint32_t need = (max_active + kUWarps - 1) / kUWarps;
    if (grid > need) grid = need;
    cudaMemsetAsync(&ctr->work, 0, sizeof(uint32_t), s);
    join_u8_kernel<<<grid, kUWarps * 32, 0, s>>>(g, c, ctr, packed, lnorm,
                                                 u8_lane_bytes(g.stride));
}

}  // namespace knng_cuda
