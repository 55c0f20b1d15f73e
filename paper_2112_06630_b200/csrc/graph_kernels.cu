// Graph-state and candidate-selection kernels (sm_100a).
//
//   init_random   KnnGraph::init_random          graph.hpp:34-67
//   load/export   KnnGraph::from_rows / rows      graph.hpp:70-93, 169-184
//   indegree      reverse_degree_ = k + in-degree graph.hpp:44,62,121-122
//   sample        select_turbo's offers           selection.hpp:282-320
//   finalize      dedup + flag_consumed + active  selection.hpp:299-302,
//                                                 graph.hpp:133-143
//
// All of these are HBM/L2-latency-bound integer work: one warp per node where
// a node's k-entry row is the unit (k <= 32: lane i owns entry i), one
// thread per edge where the edge is the unit.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace knng_cuda {

namespace {

constexpr uint32_t kSaltInit = 0x494e4954u;    // "INIT"
constexpr uint32_t kSaltSample = 0x53414d50u;  // "SAMP"
constexpr uint32_t kSaltDet = 0x44455457u;     // "DETW"

__device__ __forceinline__ uint32_t full_mask_k(uint32_t k) {
    return k >= 32 ? 0xffffffffu : ((1u << k) - 1u);
}

// Squared L2 in the reference's scalar order (l2_sq_core, distance.hpp:35-51):
// eight strided lanes, UNFUSED square-accumulate, tree
// ((0+1)+(2+3))+((4+5)+(6+7)).  Called by a full warp; the 8-lane group g
// (lanes 8g..8g+7) evaluates the pair (a_row, b_row) of its choosing and every
// lane of the group returns the distance.  (Thread-per-pair versions — 16-byte
// float loads, or dp4a over the byte copy of byte-valued data — were 1.2-1.5x
// slower: each load touches 16 bytes of a row where a group's touches a whole
// 32-byte sector.)
__device__ __forceinline__ float group8_l2_scalar(const float* __restrict__ a,
                                                  const float* __restrict__ b, uint32_t stride,
                                                  bool active) {
    const uint32_t l8 = lane_id() & 7u;
    float acc = 0.0f;
    if (active) {
#ifndef KNNG_INIT_UNROLL
#define KNNG_INIT_UNROLL 8  // measured: C5 init 56 (1) / 40 (compiler) / 34.5 (8) / 41.6 (16) ms;
                            // two pairs per group in one loop: 42.4 ms (not kept)
#endif
#if KNNG_INIT_UNROLL
#define KNNG_PRAGMA_(x) _Pragma(#x)
#define KNNG_PRAGMA(x) KNNG_PRAGMA_(x)
        KNNG_PRAGMA(unroll KNNG_INIT_UNROLL)
#endif
        for (uint32_t c = 0; c < stride; c += 8) {
            const float diff = __fsub_rn(__ldg(a + c + l8), __ldg(b + c + l8));
            acc = __fadd_rn(acc, __fmul_rn(diff, diff));
        }
    }
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 2));
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 4));
    return acc;
}

// The same distance for byte-valued data (join_u8.cu's exactness argument:
// every lane sum is an exact integer, so lane_l = |a|_l^2 + |b|_l^2 -
// 2 <a, b>_l whichever order the reference sums in) from the lane-major byte
// copy: group thread j reads bytes [8 (j + 8c), +8) of every lane segment of
// both rows (8 threads cover 64 contiguous bytes), dp4a partial dots per lane,
// an 8-thread reduce-scatter leaves lane j's dot on thread j, then the
// reference's FP32 tree.  Rows of 8 Kl bytes, Kl = 64 C.
__device__ __forceinline__ float group8_l2_u8(const uint8_t* __restrict__ a,
                                              const uint8_t* __restrict__ b,
                                              const int32_t* __restrict__ na,
                                              const int32_t* __restrict__ nb, uint32_t kl) {
    const uint32_t j = lane_id() & 7u;
    uint32_t part[8];
#pragma unroll
    for (uint32_t l = 0; l < 8; ++l) {
        uint32_t acc = 0;
        for (uint32_t o = 8 * j; o < kl; o += 64) {
            const uint2 x = __ldg(reinterpret_cast<const uint2*>(a + l * kl + o));
            const uint2 y = __ldg(reinterpret_cast<const uint2*>(b + l * kl + o));
            acc = __dp4a(x.x, y.x, acc);
            acc = __dp4a(x.y, y.y, acc);
        }
        part[l] = acc;
    }
    // reduce-scatter over the group: after the xor-4 / 2 / 1 rounds thread j
    // holds lane j's whole dot product
#pragma unroll
    for (uint32_t i = 0; i < 4; ++i) {
        const bool hi = j & 4u;
        const uint32_t send = hi ? part[i] : part[i + 4], keep = hi ? part[i + 4] : part[i];
        part[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
#pragma unroll
    for (uint32_t i = 0; i < 2; ++i) {
        const bool hi = j & 2u;
        const uint32_t send = hi ? part[i] : part[i + 2], keep = hi ? part[i + 2] : part[i];
        part[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    {
        const bool hi = j & 1u;
        const uint32_t send = hi ? part[0] : part[1], keep = hi ? part[1] : part[0];
        part[0] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
    }
    float acc = float(__ldg(na + j) + __ldg(nb + j) - 2 * int32_t(part[0]));
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 2));
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 4));
    return acc;
}

template <bool kU8>
__global__ void __launch_bounds__(256) init_random_kernel(GraphView g, uint32_t seed_lo,
                                                          uint32_t seed_hi,
                                                          const uint8_t* __restrict__ packed,
                                                          const int32_t* __restrict__ lnorm,
                                                          uint32_t kl) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (g.lo + warp >= g.hi) return;
    const uint32_t u = g.lo + warp, lane = lane_id(), k = g.k, n = g.n;
    const bool real = lane < k;
    uint32_t id = n + lane;  // placeholder, unique and never a valid id
    bool accepted = !real;
    uint32_t attempt = 0;
    const uint32_t lt = (1u << lane) - 1u;
    while (true) {
        if (!accepted) {
            const Philox4 r = philox4x32_10(u, lane, attempt, kSaltInit, seed_lo, seed_hi);
            id = bounded(r.x, n);
        }
        ++attempt;
        const uint32_t same = __match_any_sync(0xffffffffu, id);
        const uint32_t acc_mask = __ballot_sync(0xffffffffu, accepted);
        if (!accepted) {
            const uint32_t pending = ~acc_mask;
            const bool conflict = id == u || (same & acc_mask) != 0u || (same & pending & lt) != 0u;
            accepted = !conflict;
        }
        if (__all_sync(0xffffffffu, accepted)) break;
    }
    // distances: four pairs per pass, one per 8-lane group
    float mine = 0.0f;
    const float* ru = g.data + size_t(u) * g.stride;
    for (uint32_t e = 0; e < k; e += 4) {
        const uint32_t pair = e + (lane >> 3);
        const uint32_t v = __shfl_sync(0xffffffffu, id, pair & 31u);
        const bool act = pair < k;
        const uint32_t w = act ? v : u;
        const float dist =
            kU8 ? group8_l2_u8(packed + size_t(u) * 8 * kl, packed + size_t(w) * 8 * kl,
                               lnorm + size_t(u) * 8, lnorm + size_t(w) * 8, kl)
                : group8_l2_scalar(ru, g.data + size_t(w) * g.stride, g.stride, act);
        // lane (e + j) takes the result of group j (lane 8j)
        const uint32_t src = ((lane - e) & 3u) << 3;
        const float got = __shfl_sync(0xffffffffu, dist, src);
        if (lane >= e && lane < e + 4) mine = got;
    }
    uint64_t key = real ? pack_key(mine, id) : kEmptyKey;
    key = warp_sort_u64(key);
    if (real) g.keys[size_t(u) * k + lane] = key;
    const uint64_t last = __shfl_sync(0xffffffffu, key, k - 1);
    if (lane == 0) {
        g.flags[u] = full_mask_k(k);
        g.maxd[u] = key_dist(last);
    }
}

// init_random for long rows with the candidate rows bulk-copied into shared
// memory: each warp stages its node's row once and the 20 candidate rows four
// at a time (cp.async.bulk, one instruction per 4 KB row, two batches in
// flight per warp), then its four 8-lane groups evaluate the reference's
// scalar l2_sq from shared memory (same arithmetic as group8_l2_scalar, bit
// for bit).  The row-major kernel keeps ~1 KB of 32-byte loads in flight per
// warp; this one keeps up to 8 rows (30 KB for C5).
constexpr uint32_t kBulkWarpsMax = 8;

__device__ __forceinline__ uint32_t gk_su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float group8_l2_shared(const float* a, const float* b, uint32_t stride,
                                                  bool active) {
    const uint32_t l8 = lane_id() & 7u;
    float acc = 0.0f;
    if (active) {
#pragma unroll 8
        for (uint32_t c = 0; c < stride; c += 8) {
            const float diff = __fsub_rn(a[c + l8], b[c + l8]);
            acc = __fadd_rn(acc, __fmul_rn(diff, diff));
        }
    }
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 2));
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 4));
    return acc;
}

__global__ void init_random_bulk_kernel(GraphView g, uint32_t seed_lo, uint32_t seed_hi) {
    extern __shared__ __align__(128) float bulk_smem[];
    __shared__ __align__(8) unsigned long long bars[kBulkWarpsMax][2];
    const uint32_t w = threadIdx.x >> 5, lane = lane_id(), k = g.k, n = g.n;
    const uint32_t stride = g.stride, row_bytes = stride * 4;
    float* const own = bulk_smem + size_t(w) * 9 * stride;  // own row, then 2 x 4 rows
    const uint32_t warp = blockIdx.x * (blockDim.x >> 5) + w;
    const bool node = g.lo + warp < g.hi;
    const uint32_t u = node ? g.lo + warp : g.lo;
    if (lane == 0) {
        for (uint32_t b = 0; b < 2; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(gk_su32(&bars[w][b])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    if (!node) return;
    // the reference's draws: k distinct ids != u (as init_random_kernel)
    const bool real = lane < k;
    uint32_t id = n + lane;
    bool accepted = !real;
    uint32_t attempt = 0;
    const uint32_t lt = (1u << lane) - 1u;
    while (true) {
        if (!accepted) {
            const Philox4 r = philox4x32_10(u, lane, attempt, kSaltInit, seed_lo, seed_hi);
            id = bounded(r.x, n);
        }
        ++attempt;
        const uint32_t same = __match_any_sync(0xffffffffu, id);
        const uint32_t acc_mask = __ballot_sync(0xffffffffu, accepted);
        if (!accepted) {
            const uint32_t pending = ~acc_mask;
            const bool conflict = id == u || (same & acc_mask) != 0u || (same & pending & lt) != 0u;
            accepted = !conflict;
        }
        if (__all_sync(0xffffffffu, accepted)) break;
    }
    const uint32_t nb = (k + 3) / 4;
    // the ids of a batch's rows live in lanes 4 batch + j: issue reads them by shuffle
    auto issue_ids = [&](uint32_t batch) {
        uint32_t r[4];
        for (uint32_t j = 0; j < 4; ++j) r[j] = __shfl_sync(0xffffffffu, id, (4 * batch + j) & 31u);
        if (lane == 0) {
            const uint32_t b = batch & 1u, e = 4 * batch;
            const uint32_t cnt = min(4u, k - e) + (batch == 0 ? 1u : 0u);
            unsigned long long* bar = &bars[w][b];
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                             gk_su32(bar)),
                         "r"(cnt * row_bytes)
                         : "memory");
            auto copy_row = [&](float* dst, uint32_t rr) {
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], "
                    "%2, [%3];\n" ::"r"(gk_su32(dst)),
                    "l"(g.data + size_t(rr) * stride), "r"(row_bytes), "r"(gk_su32(bar))
                    : "memory");
            };
            if (batch == 0) copy_row(own, u);
            float* const buf = own + size_t(1 + 4 * b) * stride;
            for (uint32_t j = 0; j < 4 && e + j < k; ++j) copy_row(buf + size_t(j) * stride, r[j]);
        }
    };
    issue_ids(0);
    if (nb > 1) issue_ids(1);
    float mine = 0.0f;
    for (uint32_t batch = 0; batch < nb; ++batch) {
        const uint32_t b = batch & 1u, e = 4 * batch;
        const uint32_t parity = (batch >> 1) & 1u;
        asm volatile(
            "{\n .reg .pred p;\n BW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            " @!p bra BW_%=;\n}\n" ::"r"(gk_su32(&bars[w][b])),
            "r"(parity)
            : "memory");
        const uint32_t pair = e + (lane >> 3);
        const bool act = pair < k;
        const float* rv = own + size_t(1 + 4 * b + (lane >> 3)) * stride;
        const float dist = group8_l2_shared(own, rv, stride, act);
        const uint32_t src = ((lane - e) & 3u) << 3;
        const float got = __shfl_sync(0xffffffffu, dist, src);
        if (lane >= e && lane < e + 4) mine = got;
        __syncwarp();  // every group done with buffer b before it is refilled
        if (batch + 2 < nb) issue_ids(batch + 2);
    }
    uint64_t key = real ? pack_key(mine, id) : kEmptyKey;
    key = warp_sort_u64(key);
    if (real) g.keys[size_t(u) * k + lane] = key;
    const uint64_t last = __shfl_sync(0xffffffffu, key, k - 1);
    if (lane == 0) {
        g.flags[u] = full_mask_k(k);
        g.maxd[u] = key_dist(last);
    }
}

// One warp per node: rows given in any order (e.g. the reference heap order)
// -> sorted keys + flag bits.  Mirrors KnnGraph::from_rows (graph.hpp:70-93).
__global__ void __launch_bounds__(256) load_rows_kernel(GraphView g, const uint32_t* ids,
                                                        const float* dists,
                                                        const uint8_t* flags) {
    const uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (u >= g.n) return;
    const uint32_t lane = lane_id(), k = g.k;
    const bool real = lane < k;
    const size_t p = size_t(u) * k + lane;
    const uint32_t id = real ? ids[p] : 0xffffffffu;
    const uint32_t fl = real ? flags[p] : 0u;
    uint64_t key = real ? pack_key(dists[p], id) : kEmptyKey;
    key = warp_sort_u64(key);
    // flag of the entry now held by this lane: look up the original lane by id
    const uint32_t my_id = key_id(key);
    uint32_t my_flag = 0;
    for (uint32_t j = 0; j < k; ++j) {
        const uint32_t idj = __shfl_sync(0xffffffffu, id, j);
        const uint32_t flj = __shfl_sync(0xffffffffu, fl, j);
        if (real && idj == my_id) my_flag = flj;
    }
    if (real) g.keys[p] = key;
    const uint32_t mask = __ballot_sync(0xffffffffu, real && my_flag != 0u);
    const uint64_t last = __shfl_sync(0xffffffffu, key, k - 1);
    if (lane == 0) {
        g.flags[u] = mask;
        g.maxd[u] = key_dist(last);
    }
}

__global__ void export_rows_kernel(GraphView g, uint32_t* ids, float* dists, uint8_t* flags) {
    const size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t total = size_t(g.n) * g.k;
    if (e >= total) return;
    const uint64_t key = g.keys[e];
    if (ids) ids[e] = key_id(key);
    if (dists) dists[e] = key_dist(key);
    if (flags) {
        const uint32_t u = uint32_t(e / g.k), i = uint32_t(e % g.k);
        flags[e] = uint8_t((g.flags[u] >> i) & 1u);
    }
}

__global__ void indegree_kernel(GraphView g, uint32_t* indeg, const IterCounters* gate) {
    const size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= size_t(g.n) * g.k || (gate && gate->halt)) return;
    atomicAdd(indeg + key_id(g.keys[e]), 1u);
}

// select_turbo's offer (selection.hpp:296-309), concurrently: accept with
// probability cap/deg when deg > cap (deg = k + in-degree, not deduplicated,
// exactly reverse_degree); append to the target's new or old list by the
// edge's flag; once a list holds cap ids further accepts replace a uniform
// slot with reservoir probability cap/(seen) (the reference overwrites a
// uniform slot unconditionally; both keep the list a random subset).
// Duplicates are removed by finalize.
// Pair weight of candidate x offered to u in list `kind` (order-free).
__device__ __forceinline__ uint32_t det_weight(uint32_t u, uint32_t x, uint32_t kind,
                                               uint32_t seed_lo, uint32_t seed_hi) {
    return philox4x32_10(u, x, kind, kSaltDet, seed_lo, seed_hi).x;
}

__device__ __forceinline__ unsigned long long det_key(uint32_t target, uint32_t cand,
                                                      uint32_t is_new, uint32_t seed_lo,
                                                      uint32_t seed_hi) {
    return (uint64_t(det_weight(target, cand, is_new ? 1u : 2u, seed_lo, seed_hi)) << 32) | cand;
}

// turbo acceptance (selection.hpp:297-298): min(1, cap / deg), deg = k + in-degree
__device__ __forceinline__ bool accept_offer(const CandView& c, uint32_t k, const uint32_t* indeg,
                                             uint32_t target, uint32_t r_accept) {
    const uint32_t deg = k + __ldg(indeg + target);
    return !(deg > c.cap && uint64_t(r_accept) * deg >= (uint64_t(c.cap) << 32));
}

__device__ __forceinline__ void offer(const CandView& c, uint32_t k, const uint32_t* indeg,
                                      uint32_t target, uint32_t cand, uint32_t is_new,
                                      uint32_t r_accept, uint32_t r_slot, uint32_t seed_lo,
                                      uint32_t seed_hi, IterCounters* ctr) {
    if (!accept_offer(c, k, indeg, target, r_accept)) return;
    uint32_t* counter = is_new ? c.raw_new : c.raw_old;
    const uint32_t slot = atomicAdd(counter + target, 1u);
    if (c.det) {
        // every accepted offer (the expected count is <= cap; 2 cap slots);
        // which ones stay is decided on pair weights, not on arrival order:
        // an overflowing list is rebuilt by det_fix_* after this kernel
        if (slot < 2 * c.cap)
            c.raw[size_t(target) * 4 * c.cap + (is_new ? 0u : 2 * c.cap) + slot] =
                det_key(target, cand, is_new, seed_lo, seed_hi);
        else if (slot == 2 * c.cap)
            ctr->det_ovf = 1u;
        return;
    }
    uint32_t* list = c.ids + size_t(target) * 2 * c.cap + (is_new ? 0u : c.cap);
    if (slot < c.cap) {
        list[slot] = cand;
    } else {
        const uint32_t j = bounded(r_slot, slot + 1u);
        if (j < c.cap) list[j] = cand;
    }
}

// The list insertion of an accepted offer that already holds its slot (the
// reservoir rule of offer()).
__device__ __forceinline__ void place(const CandView& c, uint32_t target, uint32_t cand,
                                      uint32_t is_new, uint32_t slot, uint32_t r_slot) {
    uint32_t* list = c.ids + size_t(target) * 2 * c.cap + (is_new ? 0u : c.cap);
    if (slot < c.cap) {
        list[slot] = cand;
    } else {
        const uint32_t j = bounded(r_slot, slot + 1u);
        if (j < c.cap) list[j] = cand;
    }
}

// Non-deterministic sampling, kEdges edges per thread: every edge's in-degree
// loads, then every accepted offer's counter atomic, then the list stores, so
// a thread keeps 2 kEdges independent random accesses in flight at each step
// instead of a load -> atomic -> store chain per offer (the kernel is bound
// by their latency: ncu long-scoreboard ~90 cycles per issue).
template <uint32_t kEdges>
__global__ void __launch_bounds__(256) sample_fast_kernel(GraphView g, CandView c,
                                                          const uint32_t* __restrict__ indeg,
                                                          uint32_t seed_lo, uint32_t seed_hi,
                                                          const IterCounters* gate) {
    if (gate->halt) return;
    const size_t total = size_t(g.n) * g.k;
    const size_t e0 = (size_t(blockIdx.x) * blockDim.x) * kEdges + threadIdx.x;
    uint32_t tgt[2 * kEdges], cnd[2 * kEdges], nw[2 * kEdges], rs[2 * kEdges], slot[2 * kEdges];
    bool acc[2 * kEdges];
#pragma unroll
    for (uint32_t q = 0; q < kEdges; ++q) {
        const size_t e = e0 + size_t(q) * blockDim.x;
        acc[2 * q] = acc[2 * q + 1] = false;
        if (e >= total) continue;
        const uint32_t u = uint32_t(e / g.k), i = uint32_t(e % g.k);
        const uint32_t v = key_id(g.keys[e]);
        const uint32_t is_new = (__ldg(g.flags + u) >> i) & 1u;
        const Philox4 r = philox4x32_10(uint32_t(e), uint32_t(e >> 32), kSaltSample, 0u, seed_lo,
                                        seed_hi);
        tgt[2 * q] = u, cnd[2 * q] = v, rs[2 * q] = r.y;          // v into u
        tgt[2 * q + 1] = v, cnd[2 * q + 1] = u, rs[2 * q + 1] = r.w;  // u into v
        nw[2 * q] = nw[2 * q + 1] = is_new;
        acc[2 * q] = u >= g.lo && u < g.hi && accept_offer(c, g.k, indeg, u, r.x);
        acc[2 * q + 1] = v >= g.lo && v < g.hi && accept_offer(c, g.k, indeg, v, r.z);
    }
#pragma unroll
    for (uint32_t o = 0; o < 2 * kEdges; ++o)
        if (acc[o]) slot[o] = atomicAdd((nw[o] ? c.raw_new : c.raw_old) + tgt[o], 1u);
#pragma unroll
    for (uint32_t o = 0; o < 2 * kEdges; ++o)
        if (acc[o]) place(c, tgt[o], cnd[o], nw[o], slot[o], rs[o]);
}

__global__ void __launch_bounds__(256) sample_kernel(GraphView g, CandView c,
                                                     const uint32_t* indeg, uint32_t seed_lo,
                                                     uint32_t seed_hi, IterCounters* gate,
                                                     uint32_t det_lo, uint32_t det_hi) {
    const size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= size_t(g.n) * g.k || gate->halt) return;
    const uint32_t u = uint32_t(e / g.k), i = uint32_t(e % g.k);
    const uint32_t v = key_id(g.keys[e]);
    const uint32_t is_new = (__ldg(g.flags + u) >> i) & 1u;
    const Philox4 r = philox4x32_10(uint32_t(e), uint32_t(e >> 32), kSaltSample, 0u, seed_lo,
                                    seed_hi);
    // only lists this device owns are built; the draws are per edge, so the
    // sampled lists do not depend on how the rows are sharded
    if (u >= g.lo && u < g.hi)
        offer(c, g.k, indeg, u, v, is_new, r.x, r.y, det_lo, det_hi, gate);  // v into u
    if (v >= g.lo && v < g.hi)
        offer(c, g.k, indeg, v, u, is_new, r.z, r.w, det_lo, det_hi, gate);  // u into v
}

// Partitioned selection (multi-GPU): a shard walks only the edges
// of the rows it owns.  The forward offer (v into u) is always local; the
// reverse offer (u into v) is local when v is owned, else its acceptance is
// drawn here (the all-reduced in-degree makes deg(v) global) and an accepted
// offer becomes a record {v, u, is_new, slot draw} for owner(v) = v / chunk,
// appended to that owner's segment of `send` (segments of seg_cap records,
// counts in dst_cnt; warp-aggregated).  Edge e keeps its global index, so the
// Philox draws — and the sampled lists — do not depend on the sharding.
__global__ void __launch_bounds__(256) sample_owned_kernel(GraphView g, CandView c,
                                                           const uint32_t* indeg, uint32_t seed_lo,
                                                           uint32_t seed_hi, const IterCounters* gate,
                                                           uint32_t chunk, uint32_t* dst_cnt,
                                                           uint4* send, uint64_t seg_cap) {
    const size_t e = size_t(g.lo) * g.k + size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool in = e < size_t(g.hi) * g.k && !gate->halt;
    uint32_t dest = 0xffffffffu, v = 0, u = 0, is_new = 0;
    Philox4 r{0, 0, 0, 0};
    if (in) {
        u = uint32_t(e / g.k);
        const uint32_t i = uint32_t(e % g.k);
        v = key_id(g.keys[e]);
        is_new = (__ldg(g.flags + u) >> i) & 1u;
        r = philox4x32_10(uint32_t(e), uint32_t(e >> 32), kSaltSample, 0u, seed_lo, seed_hi);
        offer(c, g.k, indeg, u, v, is_new, r.x, r.y, 0u, 0u, nullptr);  // v into u
        if (v >= g.lo && v < g.hi)
            offer(c, g.k, indeg, v, u, is_new, r.z, r.w, 0u, 0u, nullptr);  // u into v
        else if (accept_offer(c, g.k, indeg, v, r.z))
            dest = v / chunk;
    }
    // one atomic per destination per warp
    const uint32_t peers = __match_any_sync(0xffffffffu, dest);
    const uint32_t leader = __ffs(peers) - 1u;
    uint32_t base = 0;
    if (dest != 0xffffffffu && lane_id() == leader) base = atomicAdd(dst_cnt + dest, __popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (dest != 0xffffffffu) {
        const uint32_t pos = base + __popc(peers & ((1u << lane_id()) - 1u));
        send[size_t(dest) * seg_cap + pos] = make_uint4(v, u, is_new, r.w);
    }
}

// Received reverse offers (accepted by the sender): the list insertion of
// offer(), reservoir rule included.
__global__ void apply_offers_kernel(CandView c, const uint4* recs, uint64_t count,
                                    const IterCounters* gate) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count || gate->halt) return;
    const uint4 q = recs[i];
    uint32_t* counter = q.z ? c.raw_new : c.raw_old;
    const uint32_t slot = atomicAdd(counter + q.x, 1u);
    uint32_t* list = c.ids + size_t(q.x) * 2 * c.cap + (q.z ? 0u : c.cap);
    if (slot < c.cap) {
        list[slot] = q.y;
    } else {
        const uint32_t j = bounded(q.w, slot + 1u);
        if (j < c.cap) list[j] = q.y;
    }
}

// Partial in-degree: the owned rows' edges only (the shards' partials sum to
// the in-degree, all-reduced by the caller).
__global__ void indeg_owned_kernel(GraphView g, uint32_t* indeg) {
    const size_t e = size_t(g.lo) * g.k + size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e < size_t(g.hi) * g.k) atomicAdd(indeg + key_id(g.keys[e]), 1u);
}

// Deterministic sampling, lists that received more than 2cap offers: the
// slots are reset, then every accepted offer into such a list is inserted
// again into a lock-free bounded set of the 2cap smallest keys (a key only
// replaces the current maximum; slot values only decrease, so a successful
// CAS on the scanned maximum removes the true maximum).  The result is a
// function of the set of offers, whatever the arrival order.
__global__ void det_fix_reset_kernel(GraphView g, CandView c, const IterCounters* gate) {
    const uint32_t u = g.lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= g.hi || !gate->det_ovf || gate->halt) return;
    const uint32_t cap2 = 2 * c.cap;
    unsigned long long* raw = c.raw + size_t(u) * 4 * c.cap;
    if (c.raw_new[u] > cap2)
        for (uint32_t i = 0; i < cap2; ++i) raw[i] = ~0ull;
    if (c.raw_old[u] > cap2)
        for (uint32_t i = 0; i < cap2; ++i) raw[cap2 + i] = ~0ull;
}

__device__ __forceinline__ void det_fix_offer(const CandView& c, uint32_t k, const uint32_t* indeg,
                                              uint32_t target, uint32_t cand, uint32_t is_new,
                                              uint32_t r_accept, uint32_t seed_lo,
                                              uint32_t seed_hi) {
    const uint32_t cap2 = 2 * c.cap;
    if ((is_new ? c.raw_new[target] : c.raw_old[target]) <= cap2) return;
    if (!accept_offer(c, k, indeg, target, r_accept)) return;
    const unsigned long long key = det_key(target, cand, is_new, seed_lo, seed_hi);
    unsigned long long* set = c.raw + size_t(target) * 4 * c.cap + (is_new ? 0u : cap2);
    for (;;) {
        unsigned long long mx = 0;
        uint32_t at = 0;
        for (uint32_t i = 0; i < cap2; ++i) {
            const unsigned long long v = *(volatile unsigned long long*)(set + i);
            if (v >= mx) {
                mx = v;
                at = i;
            }
        }
        if (key >= mx) return;  // not among the 2cap smallest (maxima only decrease)
        if (atomicCAS(set + at, mx, key) == mx) return;
    }
}

__global__ void __launch_bounds__(256) det_fix_sample_kernel(GraphView g, CandView c,
                                                             const uint32_t* indeg,
                                                             uint32_t seed_lo, uint32_t seed_hi,
                                                             const IterCounters* gate,
                                                             uint32_t det_lo, uint32_t det_hi) {
    const size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= size_t(g.n) * g.k || !gate->det_ovf || gate->halt) return;
    const uint32_t u = uint32_t(e / g.k), i = uint32_t(e % g.k);
    const uint32_t v = key_id(g.keys[e]);
    const uint32_t is_new = (__ldg(g.flags + u) >> i) & 1u;
    const Philox4 r = philox4x32_10(uint32_t(e), uint32_t(e >> 32), kSaltSample, 0u, seed_lo,
                                    seed_hi);
    if (u >= g.lo && u < g.hi) det_fix_offer(c, g.k, indeg, u, v, is_new, r.x, det_lo, det_hi);
    if (v >= g.lo && v < g.hi) det_fix_offer(c, g.k, indeg, v, u, is_new, r.z, det_lo, det_hi);
}

__global__ void reset_raw_kernel(CandView c, uint32_t n, const IterCounters* gate) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n || (gate && gate->halt)) return;
    c.raw_new[u] = 0u;
    c.raw_old[u] = 0u;
}

// One warp per node: clamp raw counts, dedup (within a list, first slot
// wins; across lists the copy from the edge the reference visits first wins:
// the forward edge u->x iff u < x, selection.hpp:311-317), compact, clear the
// flags of heap entries named by the new list (flag_consumed,
// graph.hpp:133-143), count the join's evaluations and list the node as
// active when nn > 0 (compute_step skips nn == 0, descent.hpp:94).
constexpr uint32_t kFinWarps = 8;
constexpr uint32_t kFinNodesPerWarp = 4;  // nodes per warp: block-level counters amortised
constexpr uint32_t kFinNodes = kFinWarps * kFinNodesPerWarp;
constexpr uint32_t kTomb = 0xffffffffu;

// Per-block accumulation (shared atomics), flushed with one global atomic per
// counter per block: the iteration counters and the active-list append are
// single global addresses, so per-node global atomics would serialise.
struct BlockCounters {
    unsigned long long evals, cands, dwords, rev;
    uint32_t nact, base;
    uint32_t act[kFinNodes];
};

__device__ __forceinline__ void init_block_counters(BlockCounters& acc) {
    if (threadIdx.x == 0) {
        acc.evals = acc.cands = acc.dwords = acc.rev = 0;
        acc.nact = 0;
    }
    __syncthreads();
}

// The join's per-node accounting (one full warp): evaluation count
// C(nn,2) + nn*no (acceptance.cpp:369-374), the size of the node's proposal
// block nn*(m + no) + m words (join.cu: one counted row per candidate), its
// entry in the active list, and one reverse-index count for every candidate
// its lists name.
__device__ __forceinline__ void join_bookkeeping(const GraphView& g, const CandView& c,
                                                 uint32_t u, uint32_t nn, uint32_t no,
                                                 BlockCounters& acc) {
    const uint32_t lane = lane_id(), m = nn + no;
    if (lane == 0) c.dsz[u] = nn ? uint64_t(nn) * (m + no) + no : 0ull;
    if (nn == 0) return;
    const uint32_t* list = c.ids + size_t(u) * 2 * c.cap;
    for (uint32_t p = lane; p < m; p += 32) {
        const uint32_t slot = p < nn ? p : c.cap + p - nn;
        const uint32_t x = list[slot];
        atomicAdd(c.revcnt + x, 1u);
        // the join's prefilter bound, gathered here once per listed candidate
        c.cmax[size_t(u) * 2 * c.cap + slot] = g.maxd[x];
    }
    if (lane == 0) {
        atomicAdd(&acc.evals, (unsigned long long)nn * (nn - 1) / 2 + (unsigned long long)nn * no);
        atomicAdd(&acc.cands, (unsigned long long)m);
        atomicAdd(&acc.dwords, (unsigned long long)nn * (m + no) + no);
        atomicAdd(&acc.rev, (unsigned long long)m);
        acc.act[atomicAdd(&acc.nact, 1u)] = u;
    }
}

// Block-collective: every thread of the block calls it once, at the end.
__device__ __forceinline__ void flush_block_counters(BlockCounters& acc, uint32_t* active,
                                                     IterCounters* ctr) {
    __syncthreads();
    if (threadIdx.x == 0) {
        if (acc.evals) atomicAdd(&ctr->evals, acc.evals);
        if (acc.cands) atomicAdd(&ctr->cands, acc.cands);
        if (acc.dwords) atomicAdd(&ctr->dwords, acc.dwords);
        if (acc.rev) atomicAdd(&ctr->rev, acc.rev);
        acc.base = acc.nact ? atomicAdd(&ctr->active, acc.nact) : 0u;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < acc.nact; i += blockDim.x) active[acc.base + i] = acc.act[i];
}

__global__ void __launch_bounds__(kFinWarps * 32, 8) finalize_kernel(GraphView g, CandView c,
                                                                  uint32_t* active,
                                                                  IterCounters* ctr) {
    __shared__ uint32_t s_new[kFinWarps][kMaxCap];
    __shared__ uint32_t s_old[kFinWarps][kMaxCap];
    __shared__ uint32_t s_hid[kFinWarps][kMaxK];
    __shared__ BlockCounters acc;
    if (ctr->halt) return;  // past termination: the graph is final
    init_block_counters(acc);
    const uint32_t w = threadIdx.x >> 5, lane = lane_id();
    const uint32_t cap = c.cap, k = g.k;
    for (uint32_t it = 0; it < kFinNodesPerWarp; ++it) {
        const uint32_t u = g.lo + (blockIdx.x * kFinNodesPerWarp + it) * kFinWarps + w;
        if (u >= g.hi) break;
        __syncwarp();  // the previous node's shared lists are no longer read
        const uint32_t nr = min(c.raw_new[u], cap), orr = min(c.raw_old[u], cap);
        const uint32_t* list = c.ids + size_t(u) * 2 * cap;
        for (uint32_t p = lane; p < nr; p += 32) s_new[w][p] = list[p];
        for (uint32_t p = lane; p < orr; p += 32) s_old[w][p] = list[cap + p];
        const uint32_t hid = lane < k ? key_id(g.keys[size_t(u) * k + lane]) : kTomb;
        s_hid[w][lane] = hid;
        const uint32_t hflags = g.flags[u];
        __syncwarp();
        // within-list duplicates: keep the first slot
        bool drop_n[2] = {false, false}, drop_o[2] = {false, false};
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h) {
            const uint32_t p = lane + 32 * h;
            if (p < nr) {
                const uint32_t x = s_new[w][p];
                for (uint32_t q = 0; q < p; ++q)
                    if (s_new[w][q] == x) { drop_n[h] = true; break; }
            }
            if (p < orr) {
                const uint32_t x = s_old[w][p];
                for (uint32_t q = 0; q < p; ++q)
                    if (s_old[w][q] == x) { drop_o[h] = true; break; }
            }
        }
        __syncwarp();
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h) {
            const uint32_t p = lane + 32 * h;
            if (p < nr && drop_n[h]) s_new[w][p] = kTomb;
            if (p < orr && drop_o[h]) s_old[w][p] = kTomb;
        }
        __syncwarp();
        // across lists
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h) {
            const uint32_t p = lane + 32 * h;
            if (p < orr && s_old[w][p] != kTomb) {
                const uint32_t x = s_old[w][p];
                for (uint32_t q = 0; q < nr; ++q) {
                    if (s_new[w][q] == x) {
                        uint32_t f_fwd = 1u;
                        for (uint32_t i = 0; i < k; ++i)
                            if (s_hid[w][i] == x) { f_fwd = (hflags >> i) & 1u; break; }
                        const bool keep_new = (u < x) ? (f_fwd != 0u) : (f_fwd == 0u);
                        if (keep_new) s_old[w][p] = kTomb; else s_new[w][q] = kTomb;
                        break;
                    }
                }
            }
        }
        __syncwarp();
        // compact both lists
        uint32_t nn = 0, no = 0;
        uint32_t* out = c.ids + size_t(u) * 2 * cap;
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h) {
            const uint32_t p = lane + 32 * h;
            const uint32_t xn = p < nr ? s_new[w][p] : kTomb;
            const uint32_t xo = p < orr ? s_old[w][p] : kTomb;
            const uint32_t mn = __ballot_sync(0xffffffffu, xn != kTomb);
            const uint32_t mo = __ballot_sync(0xffffffffu, xo != kTomb);
            const uint32_t lt = (1u << lane) - 1u;
            if (xn != kTomb) out[nn + __popc(mn & lt)] = xn;
            if (xo != kTomb) out[cap + no + __popc(mo & lt)] = xo;
            nn += __popc(mn);
            no += __popc(mo);
        }
        // flag_consumed: clear heap entries named by the final new list
        bool named = false;
        if (lane < k)
            for (uint32_t q = 0; q < nr; ++q)
                if (s_new[w][q] == hid) { named = true; break; }
        const uint32_t clear = __ballot_sync(0xffffffffu, named);
        if (lane == 0) {
            c.nc[u] = nn;
            c.oc[u] = no;
            g.flags[u] = hflags & ~clear;
        }
        join_bookkeeping(g, c, u, nn, no, acc);
    }
    flush_block_counters(acc, active, ctr);
}

// finalize with a per-warp open-addressing table instead of the O(cap^2)
// shared-memory scans above (same rules, same outputs up to the order of the
// compacted lists): every listed id is inserted once (old ids with bit 31
// set; ids < 2^31), the lowest slot holding a key wins within a list
// (atomicMin), an old id found among the new keys applies the forward-edge
// rule, and flag_consumed probes the table.  KNNG_FIN_HASH=0 builds keep the
// scan version for A/B.
#ifndef KNNG_FIN_HASH
#define KNNG_FIN_HASH 1
#endif
constexpr uint32_t kFinTab = 256;  // >= 4 kMaxCap keys at load <= 1/2
constexpr uint32_t kFinEmpty = 0xffffffffu;
constexpr uint32_t kFinDropped = 0x80000000u;  // s_first: the new copy lost to the old one

__device__ __forceinline__ uint32_t fin_hash(uint32_t key) { return (key * 0x9E3779B1u) >> 24; }

__global__ void __launch_bounds__(kFinWarps * 32, 8) finalize_hash_kernel(GraphView g, CandView c,
                                                                       uint32_t* active,
                                                                       IterCounters* ctr) {
    __shared__ uint32_t s_key[kFinWarps][kFinTab];
    __shared__ uint32_t s_first[kFinWarps][kFinTab];
    __shared__ uint32_t s_hid[kFinWarps][kMaxK];
    __shared__ BlockCounters acc;
    if (ctr->halt) return;  // past termination: the graph is final
    init_block_counters(acc);
    const uint32_t w = threadIdx.x >> 5, lane = lane_id();
    const uint32_t cap = c.cap, k = g.k;
    uint32_t* const tkey = s_key[w];
    uint32_t* const tfirst = s_first[w];
    for (uint32_t it = 0; it < kFinNodesPerWarp; ++it) {
        const uint32_t u = g.lo + (blockIdx.x * kFinNodesPerWarp + it) * kFinWarps + w;
        if (u >= g.hi) break;
        __syncwarp();  // the previous node's table is no longer read
        for (uint32_t i = lane; i < kFinTab; i += 32) {
            tkey[i] = kFinEmpty;
            tfirst[i] = kFinEmpty;
        }
        const uint32_t nr = min(c.raw_new[u], cap), orr = min(c.raw_old[u], cap);
        uint32_t* const list = c.ids + size_t(u) * 2 * cap;
        // element e: 0 / 1 new slots lane / lane + 32, 2 / 3 old slots lane / lane + 32
        uint32_t x[4], bkt[4];
        bool keep[4];
#pragma unroll
        for (uint32_t e = 0; e < 4; ++e) {
            const uint32_t p = lane + 32 * (e & 1u), cnt = e < 2 ? nr : orr;
            keep[e] = p < cnt;
            x[e] = keep[e] ? list[(e < 2 ? 0u : cap) + p] : 0u;
            bkt[e] = 0;
        }
        const uint32_t hid = lane < k ? key_id(g.keys[size_t(u) * k + lane]) : kTomb;
        s_hid[w][lane] = hid;
        const uint32_t hflags = g.flags[u];
        __syncwarp();
#pragma unroll
        for (uint32_t e = 0; e < 4; ++e) {
            if (!keep[e]) continue;
            const uint32_t key = x[e] | (e < 2 ? 0u : 0x80000000u);
            uint32_t h = fin_hash(key);
            for (;;) {
                const uint32_t prev = atomicCAS(&tkey[h], kFinEmpty, key);
                if (prev == kFinEmpty || prev == key) break;
                h = (h + 1) & (kFinTab - 1);
            }
            bkt[e] = h;
            atomicMin(&tfirst[h], lane + 32 * (e & 1u));
        }
        __syncwarp();
        // within a list the first slot wins
#pragma unroll
        for (uint32_t e = 0; e < 4; ++e)
            keep[e] = keep[e] && tfirst[bkt[e]] == lane + 32 * (e & 1u);
        __syncwarp();
        // across lists: the copy from the edge the reference visits first
        // (forward edge u -> x iff u < x, selection.hpp:311-317)
#pragma unroll
        for (uint32_t e = 2; e < 4; ++e) {
            if (!keep[e]) continue;
            const uint32_t xv = x[e];
            uint32_t h = fin_hash(xv);
            uint32_t kk;
            while ((kk = tkey[h]) != kFinEmpty && kk != xv) h = (h + 1) & (kFinTab - 1);
            if (kk != xv) continue;
            uint32_t f_fwd = 1u;
            for (uint32_t i = 0; i < k; ++i)
                if (s_hid[w][i] == xv) {
                    f_fwd = (hflags >> i) & 1u;
                    break;
                }
            const bool keep_new = (u < xv) ? (f_fwd != 0u) : (f_fwd == 0u);
            if (keep_new)
                keep[e] = false;
            else
                atomicOr(&tfirst[h], kFinDropped);
        }
        __syncwarp();
#pragma unroll
        for (uint32_t e = 0; e < 2; ++e)
            keep[e] = keep[e] && !(tfirst[bkt[e]] & kFinDropped);
        // compact both lists (slot order)
        uint32_t nn = 0, no = 0;
        const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h) {
            const uint32_t mn = __ballot_sync(0xffffffffu, keep[h]);
            const uint32_t mo = __ballot_sync(0xffffffffu, keep[2 + h]);
            if (keep[h]) list[nn + __popc(mn & lt)] = x[h];
            if (keep[2 + h]) list[cap + no + __popc(mo & lt)] = x[2 + h];
            nn += __popc(mn);
            no += __popc(mo);
        }
        // flag_consumed: clear heap entries named by the final new list
        bool named = false;
        if (hid != kTomb) {
            uint32_t h = fin_hash(hid);
            uint32_t kk;
            while ((kk = tkey[h]) != kFinEmpty && kk != hid) h = (h + 1) & (kFinTab - 1);
            named = kk == hid && !(tfirst[h] & kFinDropped);
        }
        const uint32_t clear = __ballot_sync(0xffffffffu, named);
        if (lane == 0) {
            c.nc[u] = nn;
            c.oc[u] = no;
            g.flags[u] = hflags & ~clear;
        }
        __syncwarp();  // the compacted lists, read back by other lanes
        join_bookkeeping(g, c, u, nn, no, acc);
    }
    flush_block_counters(acc, active, ctr);
}

// ---- deterministic mode ---------------------------------------------------

// Bitonic sort of 32 E keys, E per lane (element E lane + r), ascending.
template <uint32_t E, typename T>
__device__ __forceinline__ void warp_sort(T (&v)[E]) {
    const uint32_t lane = lane_id();
#pragma unroll
    for (uint32_t size = 2; size <= 32 * E; size <<= 1) {
#pragma unroll
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= E) {
#pragma unroll
                for (uint32_t r = 0; r < E; ++r) {
                    const uint32_t i = E * lane + r;
                    const T o = __shfl_xor_sync(0xffffffffu, v[r], stride / E);
                    const bool asc = (i & size) == 0, lower = (i & stride) == 0;
                    const T lo = v[r] < o ? v[r] : o, hi = v[r] < o ? o : v[r];
                    v[r] = (asc == lower) ? lo : hi;
                }
            } else {
#pragma unroll
                for (uint32_t r = 0; r < E; ++r) {
                    if (r & stride) continue;
                    const uint32_t i = E * lane + r;
                    const bool asc = (i & size) == 0;
                    const T a = v[r], b = v[r | stride];
                    if (asc ? (b < a) : (a < b)) {
                        v[r] = b;
                        v[r | stride] = a;
                    }
                }
            }
        }
    }
}

// finalize for deterministic mode, one node: both raw lists sorted by id and
// deduplicated; an id in both lists stays where the reference's first offer
// would put it (forward edge u -> x iff u < x, selection.hpp:311-317); each
// list then keeps its cap smallest pair weights, in weight order.  E = keys
// per lane of the sorts (32 E >= both raw counts).  Returns (nn, no).
template <uint32_t E>
__device__ __forceinline__ void det_lists(const GraphView& g, const CandView& c, uint32_t u,
                                          uint32_t nr, uint32_t orr, uint32_t hid,
                                          uint32_t hflags, uint32_t* s_new, uint8_t* s_kill,
                                          const uint32_t* s_hid, uint32_t seed_lo,
                                          uint32_t seed_hi, uint32_t& nn, uint32_t& no) {
    const uint32_t lane = lane_id(), cap = c.cap, k = g.k;
    const unsigned long long* raw = c.raw + size_t(u) * 4 * cap;
    uint32_t vn[E], vo[E];
#pragma unroll
    for (uint32_t r = 0; r < E; ++r) {
        const uint32_t i = E * lane + r;
        vn[r] = i < nr ? uint32_t(raw[i]) : kTomb;
        vo[r] = i < orr ? uint32_t(raw[2 * cap + i]) : kTomb;
    }
    warp_sort<E>(vn);
    warp_sort<E>(vo);
    // duplicates -> kTomb (kTomb - 1 never equals an id: ids < n < 2^31)
    auto dedup = [&](uint32_t (&v)[E]) {
        const uint32_t prev_last = __shfl_up_sync(0xffffffffu, v[E - 1], 1);
        uint32_t prev = lane == 0 ? kTomb - 1u : prev_last;
#pragma unroll
        for (uint32_t r = 0; r < E; ++r) {
            const uint32_t cur = v[r];
            if (cur == prev) v[r] = kTomb;
            prev = cur;
        }
    };
    dedup(vn);
    dedup(vo);
#pragma unroll
    for (uint32_t r = 0; r < E; ++r) {
        s_new[E * lane + r] = vn[r];
        s_kill[E * lane + r] = 0;
    }
    __syncwarp();
    // across lists: binary search of each old id in the sorted new ids
    // (matches are disjoint pairs; kills go to s_kill, s_new stays sorted)
#pragma unroll
    for (uint32_t r = 0; r < E; ++r) {
        const uint32_t x = vo[r];
        if (x == kTomb) continue;
        uint32_t lo = 0, hi = 32 * E;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (s_new[mid] < x) lo = mid + 1; else hi = mid;
        }
        if (lo < 32 * E && s_new[lo] == x) {
            uint32_t f_fwd = 1u;
            for (uint32_t i = 0; i < k; ++i)
                if (s_hid[i] == x) {
                    f_fwd = (hflags >> i) & 1u;
                    break;
                }
            const bool keep_new = (u < x) ? (f_fwd != 0u) : (f_fwd == 0u);
            if (keep_new)
                vo[r] = kTomb;
            else
                s_kill[lo] = 1;  // dropped from the new list
        }
    }
    __syncwarp();
#pragma unroll
    for (uint32_t r = 0; r < E; ++r)
        if (s_kill[E * lane + r]) vn[r] = kTomb;
    // each list: cap smallest pair weights, in weight order
    auto keep = [&](uint32_t (&v)[E], uint32_t kind, uint32_t* out, uint32_t& count) {
        unsigned long long key[E];
#pragma unroll
        for (uint32_t r = 0; r < E; ++r)
            key[r] = v[r] == kTomb
                         ? ~0ull
                         : (uint64_t(det_weight(u, v[r], kind, seed_lo, seed_hi)) << 32) | v[r];
        warp_sort<E>(key);
        uint32_t valid = 0;
#pragma unroll
        for (uint32_t r = 0; r < E; ++r) valid += key[r] != ~0ull;
#pragma unroll
        for (uint32_t o = 16; o > 0; o >>= 1) valid += __shfl_xor_sync(0xffffffffu, valid, o);
        count = min(valid, cap);
#pragma unroll
        for (uint32_t r = 0; r < E; ++r) {
            const uint32_t i = E * lane + r;
            if (i < count) out[i] = uint32_t(key[r]);
        }
    };
    uint32_t* const list = c.ids + size_t(u) * 2 * cap;
    keep(vn, 1u, list, nn);
    keep(vo, 2u, list + cap, no);
    (void)hid;
}

__global__ void __launch_bounds__(kFinWarps * 32, 4) finalize_det_kernel(GraphView g, CandView c,
                                                                      uint32_t* active,
                                                                      IterCounters* ctr,
                                                                      uint32_t seed_lo,
                                                                      uint32_t seed_hi) {
    __shared__ uint32_t s_new[kFinWarps][128];
    __shared__ uint8_t s_kill[kFinWarps][128];
    __shared__ uint32_t s_hid[kFinWarps][kMaxK];
    __shared__ BlockCounters acc;
    if (ctr->halt) return;  // past termination: the graph is final
    init_block_counters(acc);
    const uint32_t w = threadIdx.x >> 5, lane = lane_id();
    const uint32_t cap = c.cap, k = g.k;
    for (uint32_t it = 0; it < kFinNodesPerWarp; ++it) {
        const uint32_t u = g.lo + (blockIdx.x * kFinNodesPerWarp + it) * kFinWarps + w;
        if (u >= g.hi) break;
        __syncwarp();  // the previous node's shared rows are no longer read
        const uint32_t nr = min(c.raw_new[u], 2 * cap), orr = min(c.raw_old[u], 2 * cap);
        const uint32_t hid = lane < k ? key_id(g.keys[size_t(u) * k + lane]) : kTomb;
        s_hid[w][lane] = hid;
        const uint32_t hflags = g.flags[u];
        __syncwarp();
        uint32_t nn = 0, no = 0;
        const uint32_t most = max(nr, orr);
        if (most <= 32)
            det_lists<1>(g, c, u, nr, orr, hid, hflags, s_new[w], s_kill[w], s_hid[w], seed_lo,
                         seed_hi, nn, no);
        else if (most <= 64)
            det_lists<2>(g, c, u, nr, orr, hid, hflags, s_new[w], s_kill[w], s_hid[w], seed_lo,
                         seed_hi, nn, no);
        else
            det_lists<4>(g, c, u, nr, orr, hid, hflags, s_new[w], s_kill[w], s_hid[w], seed_lo,
                         seed_hi, nn, no);
        __syncwarp();
        // flag_consumed: heap entries named by the final new list
        const uint32_t* const list = c.ids + size_t(u) * 2 * cap;
        bool named = false;
        if (lane < k)
            for (uint32_t q = 0; q < nn; ++q)
                if (list[q] == hid) {
                    named = true;
                    break;
                }
        const uint32_t clear = __ballot_sync(0xffffffffu, named);
        if (lane == 0) {
            c.nc[u] = nn;
            c.oc[u] = no;
            g.flags[u] = hflags & ~clear;
        }
        join_bookkeeping(g, c, u, nn, no, acc);
    }
    flush_block_counters(acc, active, ctr);
}

// Bookkeeping only, for candidate lists supplied from outside (the
// fixed-state local-join entry): same accounting as finalize.
__global__ void __launch_bounds__(kFinWarps * 32, 8) bookkeeping_kernel(GraphView g, CandView c,
                                                                     uint32_t* active,
                                                                     IterCounters* ctr) {
    __shared__ BlockCounters acc;
    init_block_counters(acc);
    for (uint32_t it = 0; it < kFinNodesPerWarp; ++it) {
        const uint32_t u = g.lo + (blockIdx.x * kFinNodesPerWarp + it) * kFinWarps + (threadIdx.x >> 5);
        if (u < g.hi) join_bookkeeping(g, c, u, c.nc[u], c.oc[u], acc);
    }
    flush_block_counters(acc, active, ctr);
}

inline uint32_t blocks_for(size_t items, uint32_t per_block) {
    return uint32_t((items + per_block - 1) / per_block);
}

}  // namespace

void launch_init_random(const GraphView& g, uint64_t seed, cudaStream_t s, const uint8_t* packed,
                        const int32_t* lnorm) {
    if (g.hi <= g.lo) return;
    const uint32_t blocks = blocks_for(size_t(g.hi - g.lo) * 32, 256);
    // long rows: the bulk-staged kernel (KNNG_INIT_BULK=0 keeps the row-major
    // one); 9 rows of shared memory per warp
    const char* bv = getenv("KNNG_INIT_BULK");
    const size_t warp_bytes = size_t(9) * g.stride * 4;
    const uint32_t bw = uint32_t(std::min<size_t>(kBulkWarpsMax, (220u * 1024u) / warp_bytes));
    const char* bm = getenv("KNNG_INIT_BULK_MIN");
    const uint32_t bulk_min = bm ? uint32_t(atoi(bm)) : 512u;
    if (!packed && g.stride >= bulk_min && bw >= 1 && g.k <= 32 && !(bv && bv[0] == '0')) {
        static bool attr[kMaxDevices] = {};
        bool& done = attr[current_device()];
        if (!done) {
            check_launch(cudaFuncSetAttribute(init_random_bulk_kernel,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              220 * 1024));
            done = true;
        }
        const uint32_t nodes = g.hi - g.lo;
        init_random_bulk_kernel<<<(nodes + bw - 1) / bw, bw * 32, bw * warp_bytes, s>>>(
            g, uint32_t(seed), uint32_t(seed >> 32));
        return;
    }
    if (packed)
        init_random_kernel<true><<<blocks, 256, 0, s>>>(g, uint32_t(seed), uint32_t(seed >> 32),
                                                        packed, lnorm, u8_lane_bytes(g.stride));
    else
        init_random_kernel<false><<<blocks, 256, 0, s>>>(g, uint32_t(seed), uint32_t(seed >> 32),
                                                         nullptr, nullptr, 0);
}

void launch_load_rows(const GraphView& g, const uint32_t* ids, const float* dists,
                      const uint8_t* flags, cudaStream_t s) {
    load_rows_kernel<<<blocks_for(size_t(g.n) * 32, 256), 256, 0, s>>>(g, ids, dists, flags);
}

void launch_export_rows(const GraphView& g, uint32_t* ids, float* dists, uint8_t* flags,
                        cudaStream_t s) {
    export_rows_kernel<<<blocks_for(size_t(g.n) * g.k, 256), 256, 0, s>>>(g, ids, dists, flags);
}

void launch_indegree(const GraphView& g, uint32_t* indeg, cudaStream_t s,
                     const IterCounters* gate) {
    check_launch(cudaMemsetAsync(indeg, 0, sizeof(uint32_t) * g.n, s));
    indegree_kernel<<<blocks_for(size_t(g.n) * g.k, 256), 256, 0, s>>>(g, indeg, gate);
}

void launch_reset_raw(const CandView& c, uint32_t n, cudaStream_t s, const IterCounters* gate) {
    reset_raw_kernel<<<blocks_for(n, 256), 256, 0, s>>>(c, n, gate);
}

void launch_indegree_owned(const GraphView& g, uint32_t* indeg, cudaStream_t s) {
    check_launch(cudaMemsetAsync(indeg, 0, sizeof(uint32_t) * g.n, s));
    if (g.hi > g.lo)
        indeg_owned_kernel<<<blocks_for(size_t(g.hi - g.lo) * g.k, 256), 256, 0, s>>>(g, indeg);
}

void launch_sample_owned(const GraphView& g, const CandView& c, const uint32_t* indeg,
                         uint64_t seed, const IterCounters* gate, uint32_t chunk,
                         uint32_t nranks, uint32_t* dst_cnt, uint4* send, uint64_t seg_cap,
                         cudaStream_t s) {
    check_launch(cudaMemsetAsync(dst_cnt, 0, sizeof(uint32_t) * nranks, s));
    if (g.hi <= g.lo) return;
    sample_owned_kernel<<<blocks_for(size_t(g.hi - g.lo) * g.k, 256), 256, 0, s>>>(
        g, c, indeg, uint32_t(seed), uint32_t(seed >> 32), gate, chunk, dst_cnt, send, seg_cap);
}

void launch_apply_offers(const CandView& c, const uint4* recs, uint64_t count,
                         const IterCounters* gate, cudaStream_t s) {
    if (!count) return;
    apply_offers_kernel<<<uint32_t((count + 255) / 256), 256, 0, s>>>(c, recs, count, gate);
}

void launch_sample(const GraphView& g, const CandView& c, const uint32_t* indeg, uint64_t seed,
                   cudaStream_t s, IterCounters* gate, uint64_t det_seed) {
    const uint32_t blocks = blocks_for(size_t(g.n) * g.k, 256);
    const char* fv = getenv("KNNG_SAMPLE_FAST");
    if (!c.det && !(fv && fv[0] == '0')) {
        constexpr uint32_t kE = 2;
        sample_fast_kernel<kE><<<blocks_for(size_t(g.n) * g.k, 256 * kE), 256, 0, s>>>(
            g, c, indeg, uint32_t(seed), uint32_t(seed >> 32), gate);
        return;
    }
    sample_kernel<<<blocks, 256, 0, s>>>(g, c, indeg, uint32_t(seed), uint32_t(seed >> 32), gate,
                                         uint32_t(det_seed), uint32_t(det_seed >> 32));
    if (c.det && g.hi > g.lo) {
        det_fix_reset_kernel<<<blocks_for(g.hi - g.lo, 256), 256, 0, s>>>(g, c, gate);
        det_fix_sample_kernel<<<blocks, 256, 0, s>>>(g, c, indeg, uint32_t(seed),
                                                     uint32_t(seed >> 32), gate,
                                                     uint32_t(det_seed), uint32_t(det_seed >> 32));
    }
}

__global__ void iter_end_kernel(const IterCounters* cur, IterCounters* next, double threshold,
                                double recount_above) {
    next->halt = (cur->halt || cur->overflow || double(cur->changes) < threshold) ? 1u : 0u;
    if (double(cur->changes) > recount_above) next[1].recount = 1u;
}

void launch_iter_end(const IterCounters* cur, IterCounters* next, double threshold,
                     double recount_above, cudaStream_t s) {
    iter_end_kernel<<<1, 1, 0, s>>>(cur, next, threshold, recount_above);
}

__global__ void indeg_zero_kernel(uint32_t* indeg, uint32_t n, const IterCounters* gate) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n && gate->recount && !gate->halt) indeg[u] = 0u;
}

__global__ void indeg_count_kernel(GraphView g, uint32_t* indeg, const IterCounters* gate) {
    const size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= size_t(g.n) * g.k || !gate->recount || gate->halt) return;
    atomicAdd(indeg + key_id(g.keys[e]), 1u);
}

void launch_indegree_gated(const GraphView& g, uint32_t* indeg, const IterCounters* gate,
                           cudaStream_t s) {
    indeg_zero_kernel<<<blocks_for(g.n, 256), 256, 0, s>>>(indeg, g.n, gate);
    indeg_count_kernel<<<blocks_for(size_t(g.n) * g.k, 256), 256, 0, s>>>(g, indeg, gate);
}

// revcnt <- 0 unless the iteration is halted: a halted iteration must not
// clear the reverse counts an overflowed earlier iteration's rerun still needs
__global__ void zero_revcnt_kernel(uint32_t* revcnt, uint32_t n, const IterCounters* gate) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n && !gate->halt) revcnt[u] = 0u;
}

void launch_finalize(const GraphView& g, const CandView& c, uint32_t* active,
                     IterCounters* ctr, cudaStream_t s, uint64_t seed) {
    zero_revcnt_kernel<<<blocks_for(g.n, 256), 256, 0, s>>>(c.revcnt, g.n, ctr);
    if (g.hi <= g.lo) return;
    if (c.det) {
        finalize_det_kernel<<<blocks_for(g.hi - g.lo, kFinNodes), kFinWarps * 32, 0, s>>>(
            g, c, active, ctr, uint32_t(seed), uint32_t(seed >> 32));
        return;
    }
#if KNNG_FIN_HASH
    finalize_hash_kernel<<<blocks_for(g.hi - g.lo, kFinNodes), kFinWarps * 32, 0, s>>>(g, c, active,
                                                                                       ctr);
#else
    finalize_kernel<<<blocks_for(g.hi - g.lo, kFinNodes), kFinWarps * 32, 0, s>>>(g, c, active,
                                                                                  ctr);
#endif
}

void launch_bookkeeping(const GraphView& g, const CandView& c, uint32_t* active,
                        IterCounters* ctr, cudaStream_t s) {
    check_launch(cudaMemsetAsync(c.revcnt, 0, sizeof(uint32_t) * g.n, s));
    if (g.hi <= g.lo) return;
    bookkeeping_kernel<<<blocks_for(g.hi - g.lo, kFinNodes), kFinWarps * 32, 0, s>>>(g, c, active,
                                                                                     ctr);
}

}  // namespace knng_cuda
