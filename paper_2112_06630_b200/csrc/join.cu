// The local join (compute_step, reference descent.hpp:82-153) on sm_100a.
//
// One CTA owns one active node u at a time (persistent grid, nodes handed out
// by an atomic work counter).  For u's new list N (nn ids) and old list O (no
// ids) it
//   1. evaluates every new x new unordered pair and every new x old pair
//      (the same C(nn,2) + nn*no evaluations as compute_step) into a
//      distance matrix D in shared memory, and then
//   2. for every candidate t in N u O gathers the partners whose distance
//      beats t's cached row maximum (the stale-upwards prefilter of
//      descent.hpp:97-102,134-147) and merges them into t's bounded sorted
//      row under t's lock with try_insert's semantics (graph.hpp:116-129):
//      strict improvement over the current maximum, id dedup, evict the max.
//
// Distances are bit-identical to the reference's compiled kernels.  The
// reference sums (a_j - b_j)^2 in eight strided lanes (lane l owns elements
// 8c + l) and reduces them as ((0+1)+(2+3))+((4+5)+(6+7)) (distance.hpp:29-51).
// Pairs that fall into a full 5x5 or triangular tile (block_core /
// tri_core5) are accumulated with a fused multiply-add, the rest (remainder
// rows of mutual_block_distances, partial new x old tiles) unfused
// (pinned in tests/test_oracle_pins.py).  Here a group of 8
// threads is one pair-tile and thread l8 of the group is reference lane l8:
// it accumulates elements 8c + l8 of a 4x4 pair tile with the path of each
// pair, and the group combines lanes with shfl_xor 1, 2, 4 — exactly the
// reference tree — as a reduce-scatter (14 shuffles for 16 pairs).
#include "kernels.cuh"

namespace knng_cuda {

namespace {

constexpr uint32_t kTileR = 4;
constexpr uint32_t kTileC = 4;
constexpr uint32_t kTilePairs = kTileR * kTileC;

enum TileMode : int { kFused = 0, kUnfused = 1, kMixed = 2 };

template <int MODE>
__device__ __forceinline__ void tile_accumulate(const float* const (&pa)[kTileR],
                                                const float* const (&pb)[kTileC],
                                                uint32_t stride, uint32_t l8,
                                                float (&acc)[kTilePairs], uint32_t fused_mask) {
#pragma unroll 2
    for (uint32_t c = l8; c < stride; c += 8) {
        float a[kTileR], b[kTileC];
#pragma unroll
        for (uint32_t x = 0; x < kTileR; ++x) a[x] = __ldg(pa[x] + c);
#pragma unroll
        for (uint32_t y = 0; y < kTileC; ++y) b[y] = __ldg(pb[y] + c);
#pragma unroll
        for (uint32_t x = 0; x < kTileR; ++x) {
#pragma unroll
            for (uint32_t y = 0; y < kTileC; ++y) {
                const uint32_t p = x * kTileC + y;
                const float diff = __fsub_rn(a[x], b[y]);
                if (MODE == kFused) {
                    acc[p] = __fmaf_rn(diff, diff, acc[p]);
                } else if (MODE == kUnfused) {
                    acc[p] = __fadd_rn(acc[p], __fmul_rn(diff, diff));
                } else {
                    const float fused = __fmaf_rn(diff, diff, acc[p]);
                    const float plain = __fadd_rn(acc[p], __fmul_rn(diff, diff));
                    acc[p] = ((fused_mask >> p) & 1u) ? fused : plain;
                }
            }
        }
    }
}

// Reduce-scatter of 16 per-lane partial sums over the 8 lanes of a group in
// the reference's tree order.  Lane l8 = b0 + 2 b1 + 4 b2 ends with the full
// sums of pairs base, base+1 where base = 8 b0 + 4 b1 + 2 b2.
__device__ __forceinline__ void group_reduce(const float (&acc)[kTilePairs], uint32_t l8,
                                             float (&out)[2]) {
    const bool b0 = l8 & 1u, b1 = (l8 >> 1) & 1u, b2 = (l8 >> 2) & 1u;
    float r8[8];
#pragma unroll
    for (uint32_t j = 0; j < 8; ++j) {
        const float send = b0 ? acc[j] : acc[8 + j];
        const float keep = b0 ? acc[8 + j] : acc[j];
        r8[j] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 1));
    }
    float r4[4];
#pragma unroll
    for (uint32_t j = 0; j < 4; ++j) {
        const float send = b1 ? r8[j] : r8[4 + j];
        const float keep = b1 ? r8[4 + j] : r8[j];
        r4[j] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 2));
    }
#pragma unroll
    for (uint32_t j = 0; j < 2; ++j) {
        const float send = b2 ? r4[j] : r4[2 + j];
        const float keep = b2 ? r4[2 + j] : r4[j];
        out[j] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 4));
    }
}

// Warp-wide bounded insert into a sorted row held one key per lane (lanes
// >= k hold kEmptyKey).  try_insert semantics (graph.hpp:116-129).
__device__ __forceinline__ bool warp_try_insert(uint64_t& key, uint32_t& flags, uint32_t k,
                                                float dist, uint32_t cand) {
    const uint32_t lane = lane_id();
    const uint64_t max_key = __shfl_sync(0xffffffffu, key, k - 1);
    if (!(dist < key_dist(max_key))) return false;
    if (__ballot_sync(0xffffffffu, lane < k && key_id(key) == cand)) return false;
    const uint64_t nk = pack_key(dist, cand);
    const uint32_t pos = __popc(__ballot_sync(0xffffffffu, lane < k && key < nk));
    const uint64_t up = __shfl_up_sync(0xffffffffu, key, 1);
    if (lane < k) key = lane < pos ? key : (lane == pos ? nk : up);
    const uint32_t low = (1u << pos) - 1u;
    const uint32_t kmask = k >= 32 ? 0xffffffffu : ((1u << k) - 1u);
    flags = ((flags & low) | (1u << pos) | ((flags & ~low) << 1)) & kmask;
    return true;
}

struct JoinShared {
    uint32_t node;
    uint32_t nn, no;
    unsigned long long changes;
};

template <uint32_t kThreads, bool kDistOnly>
__global__ void __launch_bounds__(kThreads) join_kernel(GraphView g, CandView c,
                                                        const uint32_t* __restrict__ active,
                                                        uint32_t* work_counter,
                                                        IterCounters* ctr,
                                                        const uint64_t* offsets, float* out) {
    constexpr uint32_t kWarps = kThreads / 32;
    constexpr uint32_t kGroups = kThreads / 8;
    extern __shared__ float s_D[];               // nn x m, m = nn + no (<= cap x 2cap)
    __shared__ uint32_t s_ids[2 * kMaxCap];
    __shared__ JoinShared sh;

    const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    const uint32_t group = tid >> 3, l8 = tid & 7u;
    const uint32_t k = g.k, cap = c.cap, stride = g.stride;
    const uint32_t n_active = ctr->active;
    if (tid == 0) sh.changes = 0;

    while (true) {
        __syncthreads();
        if (tid == 0) {
            const uint32_t a = atomicAdd(work_counter, 1u);
            sh.node = a < n_active ? active[a] : 0xffffffffu;
            if (a < n_active) {
                sh.nn = c.nc[sh.node];
                sh.no = c.oc[sh.node];
            }
        }
        __syncthreads();
        const uint32_t u = sh.node;
        if (u == 0xffffffffu) break;
        const uint32_t nn = sh.nn, no = sh.no, m = nn + no;
        const uint32_t* list = c.ids + size_t(u) * 2 * cap;
        for (uint32_t i = tid; i < nn; i += kThreads) s_ids[i] = list[i];
        for (uint32_t i = tid; i < no; i += kThreads) s_ids[nn + i] = list[cap + i];
        __syncthreads();

        // ---- 1. distances -------------------------------------------------
        const uint32_t full_n = nn - nn % 5, full_o = no - no % 5;
        const uint32_t rb = (nn + kTileR - 1) / kTileR, ob = (no + kTileC - 1) / kTileC;
        const uint32_t t_nn = rb * (rb + 1) / 2, t_all = t_nn + rb * ob;
        for (uint32_t t = group; t < t_all; t += kGroups) {
            uint32_t bi, col0;
            bool col_new;
            if (t < t_nn) {
                uint32_t tt = t;
                bi = 0;
                while (tt >= rb - bi) {
                    tt -= rb - bi;
                    ++bi;
                }
                col0 = (bi + tt) * kTileC;
                col_new = true;
            } else {
                const uint32_t tt = t - t_nn;
                bi = tt / ob;
                col0 = nn + (tt % ob) * kTileC;
                col_new = false;
            }
            const uint32_t row0 = bi * kTileR;
            const float* pa[kTileR];
            const float* pb[kTileC];
            uint32_t valid_mask = 0, fused_mask = 0;
#pragma unroll
            for (uint32_t x = 0; x < kTileR; ++x) {
                const uint32_t r = row0 + x;
                pa[x] = g.data + size_t(s_ids[r < nn ? r : 0]) * stride;
            }
#pragma unroll
            for (uint32_t y = 0; y < kTileC; ++y) {
                const uint32_t cc = col0 + y;
                const bool cvalid = col_new ? cc < nn : cc < m;
                pb[y] = g.data + size_t(s_ids[cvalid ? cc : 0]) * stride;
                const bool cfused = col_new ? cc < full_n : (cc - nn) < full_o;
#pragma unroll
                for (uint32_t x = 0; x < kTileR; ++x) {
                    const uint32_t r = row0 + x;
                    const bool valid = r < nn && cvalid && (!col_new || cc > r);
                    const bool fused = r < full_n && cfused;
                    valid_mask |= uint32_t(valid) << (x * kTileC + y);
                    fused_mask |= uint32_t(fused) << (x * kTileC + y);
                }
            }
            float acc[kTilePairs];
#pragma unroll
            for (uint32_t p = 0; p < kTilePairs; ++p) acc[p] = 0.0f;
            if ((fused_mask & valid_mask) == valid_mask)
                tile_accumulate<kFused>(pa, pb, stride, l8, acc, fused_mask);
            else if ((fused_mask & valid_mask) == 0u)
                tile_accumulate<kUnfused>(pa, pb, stride, l8, acc, fused_mask);
            else
                tile_accumulate<kMixed>(pa, pb, stride, l8, acc, fused_mask);
            float res[2];
            group_reduce(acc, l8, res);
            const uint32_t base = 8u * (l8 & 1u) + 4u * ((l8 >> 1) & 1u) + 2u * ((l8 >> 2) & 1u);
#pragma unroll
            for (uint32_t j = 0; j < 2; ++j) {
                const uint32_t p = base + j;
                if ((valid_mask >> p) & 1u) {
                    const uint32_t x = p / kTileC, y = p % kTileC;
                    s_D[(row0 + x) * m + col0 + y] = res[j];
                }
            }
        }
        __syncthreads();

        if (kDistOnly) {
            float* dst = out + offsets[u];
            for (uint32_t e = tid; e < nn * m; e += kThreads) {
                const uint32_t i = e / m, j = e % m;
                if (j >= nn || j > i) dst[e] = s_D[e];
            }
            continue;
        }

        // ---- 2. proposals + locked merges -----------------------------------
        for (uint32_t r = warp; r < m; r += kWarps) {
            const uint32_t t = s_ids[r];
            const float mx = ld_cg_f32(g.maxd + t);
            const uint32_t P = r < nn ? (nn - 1 + no) : nn;
            auto partner = [&](uint32_t q, float& dist, uint32_t& cand) {
                if (r < nn) {
                    if (q + 1 < nn) {
                        const uint32_t j = q < r ? q : q + 1;
                        dist = r < j ? s_D[r * m + j] : s_D[j * m + r];
                        cand = s_ids[j];
                    } else {
                        const uint32_t jj = q + 1;  // nn + (q - (nn - 1))
                        dist = s_D[r * m + jj];
                        cand = s_ids[jj];
                    }
                } else {
                    dist = s_D[q * m + r];
                    cand = s_ids[q];
                }
            };
            bool any = false;
            for (uint32_t q0 = 0; q0 < P; q0 += 32) {
                const uint32_t q = q0 + lane;
                float dist = 0.0f;
                uint32_t cand = 0;
                if (q < P) partner(q, dist, cand);
                any |= __ballot_sync(0xffffffffu, q < P && dist < mx) != 0u;
            }
            if (!any) continue;

            if (lane == 0) {
                while (atomicCAS(g.locks + t, 0u, 1u) != 0u) __nanosleep(20);
                __threadfence();
            }
            __syncwarp();
            uint64_t key = lane < k ? ld_cg_u64(g.keys + size_t(t) * k + lane) : kEmptyKey;
            uint32_t flags = ld_cg_u32(g.flags + t);
            uint32_t inserted = 0;
            for (uint32_t q0 = 0; q0 < P; q0 += 32) {
                const uint32_t q = q0 + lane;
                float dist = 0.0f;
                uint32_t cand = 0;
                if (q < P) partner(q, dist, cand);
                uint32_t pass = __ballot_sync(0xffffffffu, q < P && dist < mx);
                while (pass) {
                    const uint32_t src = __ffs(pass) - 1u;
                    pass &= pass - 1u;
                    const float dd = __shfl_sync(0xffffffffu, dist, src);
                    const uint32_t cc = __shfl_sync(0xffffffffu, cand, src);
                    inserted += warp_try_insert(key, flags, k, dd, cc) ? 1u : 0u;
                }
            }
            if (inserted) {
                if (lane < k) st_cg_u64(g.keys + size_t(t) * k + lane, key);
                const uint64_t last = __shfl_sync(0xffffffffu, key, k - 1);
                if (lane == 0) {
                    st_cg_u32(g.flags + t, flags);
                    st_cg_f32(g.maxd + t, key_dist(last));
                }
            }
            __threadfence();
            __syncwarp();
            if (lane == 0) {
                atomicExch(g.locks + t, 0u);
                if (inserted) atomicAdd(&sh.changes, (unsigned long long)inserted);
            }
        }
    }
    __syncthreads();
    if (!kDistOnly && tid == 0 && sh.changes) atomicAdd(&ctr->changes, sh.changes);
}

uint32_t g_sm_count = 0;

uint32_t sm_count() {
    if (!g_sm_count) {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        g_sm_count = v > 0 ? uint32_t(v) : 148u;
    }
    return g_sm_count;
}

template <uint32_t kThreads, bool kDistOnly>
void launch_join_impl(const GraphView& g, const CandView& c, const uint32_t* active,
                      uint32_t max_active, IterCounters* ctr, const uint64_t* offsets, float* out,
                      uint32_t* work_counter, cudaStream_t s) {
    const size_t smem = join_smem_bytes(c.cap);
    auto kern = join_kernel<kThreads, kDistOnly>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, int(kThreads), smem);
    if (per_sm < 1) per_sm = 1;
    uint32_t grid = sm_count() * uint32_t(per_sm);
    if (grid > max_active) grid = max_active;
    if (grid == 0) return;
    cudaMemsetAsync(work_counter, 0, sizeof(uint32_t), s);
    kern<<<grid, kThreads, smem, s>>>(g, c, active, work_counter, ctr, offsets, out);
}

}  // namespace

size_t join_smem_bytes(uint32_t cap) { return size_t(cap) * 2 * cap * sizeof(float); }

// The work counter lives in the IterCounters' padding word.
void launch_join(const GraphView& g, const CandView& c, const uint32_t* active,
                 uint32_t max_active, IterCounters* ctr, cudaStream_t s) {
    uint32_t* wc = &ctr->pad;
    if (c.cap <= 32)
        launch_join_impl<128, false>(g, c, active, max_active, ctr, nullptr, nullptr, wc, s);
    else
        launch_join_impl<256, false>(g, c, active, max_active, ctr, nullptr, nullptr, wc, s);
}

void launch_join_distances(const GraphView& g, const CandView& c, const uint32_t* active,
                           uint32_t max_active, const uint64_t* offsets, float* out,
                           cudaStream_t s, IterCounters* ctr) {
    uint32_t* wc = &ctr->pad;
    if (c.cap <= 32)
        launch_join_impl<128, true>(g, c, active, max_active, ctr, offsets, out, wc, s);
    else
        launch_join_impl<256, true>(g, c, active, max_active, ctr, offsets, out, wc, s);
}

}  // namespace knng_cuda
