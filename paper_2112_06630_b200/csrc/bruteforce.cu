// Exact K-NNG on the GPU — the measurement oracle for recall at scale
// (brute_force_knng, reference oracle.hpp:92-127).
//
// Stage 1 (bf_filter): CTA tiles of 64 queries x 64 candidates, difference
// form (q - c)^2 accumulated in FP32 with a 4x4 register tile per thread,
// streaming 32-dimension slabs through shared memory.  Every tile's survivors
// (below the query's current 64th-best distance) are merged into a sorted
// per-query list of the 64 best (distance, id) keys held in shared memory.
// Stage 2 (bf_rerank): the 64 survivors per query are re-evaluated in FP64 in
// the reference's order (8 lanes over the true d, fused square-accumulate as
// the reference's compiled double loop does, tree reduction, tail;
// l2_sq_double, oracle.hpp:50-66) and ranked by (distance, id) — the
// reference's total order (oracle.hpp:71-76) — keeping the first k.  With
// k <= 32 the 32+ spare slots absorb FP32 rounding, so the result is
// index-exact (checked against the CPU brute force in tests).
#include "kernels.cuh"

namespace knng_cuda {

namespace {

constexpr uint32_t kQB = 64;     // queries per CTA
constexpr uint32_t kCB = 64;     // candidates per tile
constexpr uint32_t kDK = 32;     // dimensions per smem slab
constexpr uint32_t kK2 = 64;     // filtered list length per query
constexpr uint32_t kBfThreads = 256;

struct BfShared {
    float q[kDK][kQB + 4];
    float c[kDK][kCB + 4];
    uint64_t top[kQB][kK2];
    uint64_t buf[kQB][kCB];
    uint32_t bufcnt[kQB];
    float thr[kQB];
};

// Insert key nk into a sorted 64-entry list held two per lane (entry lane and
// 32 + lane); the largest entry falls off.
__device__ __forceinline__ void warp_insert64(uint64_t& lo, uint64_t& hi, uint64_t nk) {
    const uint32_t lane = lane_id();
    const uint32_t pos = __popc(__ballot_sync(0xffffffffu, lo < nk)) +
                         __popc(__ballot_sync(0xffffffffu, hi < nk));
    const uint64_t lo_up = __shfl_up_sync(0xffffffffu, lo, 1);
    const uint64_t hi_up = __shfl_up_sync(0xffffffffu, hi, 1);
    const uint64_t lo_last = __shfl_sync(0xffffffffu, lo, 31);
    const uint32_t ehi = 32 + lane;
    const uint64_t hi_prev = lane == 0 ? lo_last : hi_up;
    const uint64_t new_hi = ehi < pos ? hi : (ehi == pos ? nk : hi_prev);
    const uint64_t new_lo = lane < pos ? lo : (lane == pos ? nk : lo_up);
    lo = new_lo;
    hi = new_hi;
}

__global__ void __launch_bounds__(kBfThreads) bf_filter_kernel(const float* __restrict__ data,
                                                               uint32_t n, uint32_t stride,
                                                               const uint32_t* __restrict__ queries,
                                                               uint32_t nq,
                                                               uint64_t* __restrict__ out_top) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BfShared& sh = *reinterpret_cast<BfShared*>(smem_raw);
    const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    const uint32_t ty = tid >> 4, tx = tid & 15u;
    const uint32_t q0 = blockIdx.x * kQB;

    for (uint32_t i = tid; i < kQB * kK2; i += kBfThreads) (&sh.top[0][0])[i] = kEmptyKey;
    for (uint32_t i = tid; i < kQB; i += kBfThreads) {
        sh.bufcnt[i] = 0;
        sh.thr[i] = __int_as_float(0x7f800000);  // +inf
    }
    // query ids of my rows
    uint32_t qid[4];
#pragma unroll
    for (uint32_t x = 0; x < 4; ++x) {
        const uint32_t qi = q0 + 4 * ty + x;
        qid[x] = qi < nq ? queries[qi] : 0xffffffffu;
    }
    __syncthreads();

    for (uint32_t c0 = 0; c0 < n; c0 += kCB) {
        float acc[16];
#pragma unroll
        for (uint32_t p = 0; p < 16; ++p) acc[p] = 0.0f;
        for (uint32_t k0 = 0; k0 < stride; k0 += kDK) {
            // stage 64 x 32 slabs, transposed: thread loads 8 floats of one row
            {
                const uint32_t r = tid >> 2, part = (tid & 3u) * 8;
                const uint32_t qi = q0 + r;
                const uint32_t qrow = qi < nq ? queries[qi] : 0u;
                const uint32_t crow = c0 + r < n ? c0 + r : 0u;
#pragma unroll
                for (uint32_t j = 0; j < 8; ++j) {
                    const uint32_t dd = k0 + part + j;
                    const bool in = dd < stride;
                    sh.q[part + j][r] = in ? __ldg(data + size_t(qrow) * stride + dd) : 0.0f;
                    sh.c[part + j][r] = in ? __ldg(data + size_t(crow) * stride + dd) : 0.0f;
                }
            }
            __syncthreads();
#pragma unroll 8
            for (uint32_t dd = 0; dd < kDK; ++dd) {
                const float4 a = *reinterpret_cast<const float4*>(&sh.q[dd][4 * ty]);
                const float4 b = *reinterpret_cast<const float4*>(&sh.c[dd][4 * tx]);
                const float av[4] = {a.x, a.y, a.z, a.w};
                const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                for (uint32_t x = 0; x < 4; ++x)
#pragma unroll
                    for (uint32_t y = 0; y < 4; ++y) {
                        const float diff = av[x] - bv[y];
                        acc[x * 4 + y] = fmaf(diff, diff, acc[x * 4 + y]);
                    }
            }
            __syncthreads();
        }
        // survivors into per-query buffers
#pragma unroll
        for (uint32_t x = 0; x < 4; ++x) {
            const uint32_t ql = 4 * ty + x;
            const float thr = sh.thr[ql];
#pragma unroll
            for (uint32_t y = 0; y < 4; ++y) {
                const uint32_t cid = c0 + 4 * tx + y;
                const float dist = acc[x * 4 + y];
                if (qid[x] != 0xffffffffu && cid < n && cid != qid[x] && dist <= thr) {
                    const uint32_t slot = atomicAdd(&sh.bufcnt[ql], 1u);
                    sh.buf[ql][slot] = pack_key(dist, cid);
                }
            }
        }
        __syncthreads();
        // merge: one warp per query
        for (uint32_t ql = warp; ql < kQB; ql += kBfThreads / 32) {
            const uint32_t cnt = sh.bufcnt[ql];
            if (cnt == 0) continue;
            uint64_t lo = sh.top[ql][lane], hi = sh.top[ql][32 + lane];
            for (uint32_t i = 0; i < cnt; ++i) {
                const uint64_t nk = sh.buf[ql][i];
                const uint64_t last = __shfl_sync(0xffffffffu, hi, 31);
                if (nk < last) warp_insert64(lo, hi, nk);
            }
            sh.top[ql][lane] = lo;
            sh.top[ql][32 + lane] = hi;
            const uint64_t last = __shfl_sync(0xffffffffu, hi, 31);
            if (lane == 0) {
                sh.bufcnt[ql] = 0;
                sh.thr[ql] = last == kEmptyKey ? __int_as_float(0x7f800000) : key_dist(last);
            }
        }
        __syncthreads();
    }
    for (uint32_t i = tid; i < kQB * kK2; i += kBfThreads) {
        const uint32_t ql = i / kK2;
        if (q0 + ql < nq) out_top[size_t(q0 + ql) * kK2 + (i % kK2)] = (&sh.top[0][0])[i];
    }
}

// One warp per query: FP64 re-evaluation of the 64 survivors in the
// reference's accumulation order, then rank by (distance, id).
__global__ void __launch_bounds__(256) bf_rerank_kernel(const float* __restrict__ data,
                                                        uint32_t stride, uint32_t d, uint32_t k,
                                                        const uint32_t* __restrict__ queries,
                                                        uint32_t nq, const uint64_t* top,
                                                        uint32_t* out_ids, double* out_dists) {
    const uint32_t qi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (qi >= nq) return;
    const uint32_t lane = lane_id(), l8 = lane & 7u, grp = lane >> 3;
    const uint32_t q = queries[qi];
    const float* rq = data + size_t(q) * stride;
    double mine[2] = {0.0, 0.0};
    uint32_t my_id[2];
    my_id[0] = key_id(top[size_t(qi) * kK2 + lane]);
    my_id[1] = key_id(top[size_t(qi) * kK2 + 32 + lane]);
    const uint32_t chunks = d / 8;
    for (uint32_t e0 = 0; e0 < kK2; e0 += 4) {
        const uint32_t e = e0 + grp;
        const uint32_t cid = __shfl_sync(0xffffffffu, my_id[e >> 5], e & 31u);
        double acc = 0.0;
        if (cid != 0xffffffffu) {
            const float* rc = data + size_t(cid) * stride;
            for (uint32_t c = 0; c < chunks; ++c) {
                const double diff = double(rq[8 * c + l8]) - double(rc[8 * c + l8]);
                acc = __fma_rn(diff, diff, acc);
            }
        }
        double s1 = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));
        double s2 = __dadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, 2));
        double s3 = __dadd_rn(s2, __shfl_xor_sync(0xffffffffu, s2, 4));
        double tail = 0.0;
        if (cid != 0xffffffffu) {
            const float* rc = data + size_t(cid) * stride;
            for (uint32_t j = chunks * 8; j < d; ++j) {
                const double diff = double(rq[j]) - double(rc[j]);
                tail = __fma_rn(diff, diff, tail);
            }
        }
        const double total = cid == 0xffffffffu ? __longlong_as_double(0x7ff0000000000000ll)
                                                : __dadd_rn(s3, tail);
        // entry e's owner lane (e & 31), slot e >> 5, takes group grp's result
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) {
            const double v = __shfl_sync(0xffffffffu, total, j * 8);
            const uint32_t ej = e0 + j;
            if ((ej & 31u) == lane) mine[ej >> 5] = v;
        }
    }
    // rank by (dist, id)
#pragma unroll
    for (uint32_t h = 0; h < 2; ++h) {
        uint32_t rank = 0;
        for (uint32_t src = 0; src < 32; ++src) {
#pragma unroll
            for (uint32_t h2 = 0; h2 < 2; ++h2) {
                const double od = __shfl_sync(0xffffffffu, mine[h2], src);
                const uint32_t oi = __shfl_sync(0xffffffffu, my_id[h2], src);
                rank += (od < mine[h] || (od == mine[h] && oi < my_id[h])) ? 1u : 0u;
            }
        }
        if (rank < k && my_id[h] != 0xffffffffu) {
            out_ids[size_t(qi) * k + rank] = my_id[h];
            if (out_dists) out_dists[size_t(qi) * k + rank] = mine[h];
        }
    }
}

__global__ void iota_kernel(uint32_t* p, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = i;
}

}  // namespace

void launch_bruteforce_queries(const float* data, uint32_t n, uint32_t d, uint32_t stride,
                               uint32_t k, const uint32_t* queries, uint32_t nq,
                               uint64_t* scratch_top, uint32_t* out_ids, double* out_dists,
                               cudaStream_t s) {
    const size_t smem = sizeof(BfShared);
    cudaFuncSetAttribute(bf_filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    bf_filter_kernel<<<(nq + kQB - 1) / kQB, kBfThreads, smem, s>>>(data, n, stride, queries, nq,
                                                                    scratch_top);
    bf_rerank_kernel<<<(nq * 32 + 255) / 256, 256, 0, s>>>(data, stride, d, k, queries, nq,
                                                           scratch_top, out_ids, out_dists);
}

void launch_iota(uint32_t* p, uint32_t n, cudaStream_t s) {
    iota_kernel<<<(n + 255) / 256, 256, 0, s>>>(p, n);
}

size_t bruteforce_scratch_keys(uint32_t nq) { return size_t(nq) * kK2; }

}  // namespace knng_cuda
