// The local join's distance stage with tiles aligned to the reference's
// 5-blocking (compute_step, reference descent.hpp:82-153; block_core /
// tri_core5 and the flexible remainder paths, distance.hpp:134-190).
//
// join.cu's kernel cuts a node's pair matrix into 8 x 8 tiles; because a tile
// must be wholly fused or wholly unfused (the reference's compiler contracts
// multiply-add only inside full 5 x 5 / triangular tiles) it
// permutes rows and columns into padded slot groups, and for mid-size lists
// (nn = 5..20 new, 20..40 old candidates) only a quarter to a third of the
// computed pair slots are live.  Here a tile is 5 rows x 10 columns (two
// independent 5-column blocks), so the reference's own block boundaries are
// tile boundaries:
//   F  (fused)    new rows [5i, 5i + 5) x two 5-blocks out of
//                 {new blocks j >= i (j == i: the triangle)} ++ {full old blocks}
//   U  (unfused)  the nn % 5 leftover new rows x every column, 10 at a time
//   U2 (unfused)  the no % 5 leftover old candidates (as rows) x the fused
//                 new candidates, 10 at a time
// A node's candidates keep their list order as slots (new, then old), with no
// padding inside a node or between the nodes of a batch.  nn = 7, no = 23:
// 3 F + 3 U + 1 U2 tiles of 50 pairs against ten 8 x 8 tiles.
//
// Everything else is join.cu's design: persistent CTAs of 16 groups of 8
// lanes (thread l8 = reference lane l8, packed FFMA2 arithmetic, the
// reference's reduction tree as a reduce-scatter), batches of nodes formed one
// ahead, candidate rows staged by cp.async through a 3-stage ring of
// 32-float slabs (pass mode) or once per batch (resident mode), proposals
// prefiltered against each endpoint's row maximum and compacted into the
// node's proposal block.  Distances are bit-identical to join.cu's and the
// reference's (tests/test_gpu_parity.py runs both kernels against the oracle).
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"
#include "tile_math.cuh"

namespace knng_cuda {

namespace {

constexpr uint32_t kThreads = 128;  // 16 groups of 8 lanes
constexpr uint32_t kGroups = kThreads / 8;
constexpr uint32_t kSlab = 32;      // floats per row per ring stage
constexpr uint32_t kStages = 3;
// Ring rows are kPitch floats apart: 36 puts rows r and r + 10 (the column
// blocks of the four tiles a warp usually runs) 8 banks apart, and rows r and
// r + 5 20 banks apart, so the groups' 8-bank reads do not collide.
constexpr uint32_t kPitch = 36;
#ifndef KNNG_T5_PASSBLK
#define KNNG_T5_PASSBLK 14
#endif
constexpr uint32_t kPassBlk = KNNG_T5_PASSBLK;  // 8-slot blocks one pass may stage
constexpr uint32_t kRingRows = kPassBlk * 8;
constexpr uint32_t kMaxBatch = 8;
constexpr uint32_t kSlotTab = 320;  // batch slots
constexpr uint32_t kBlkTab = kSlotTab / 8;
constexpr uint32_t kMaxTiles = 384;
constexpr uint32_t kDeadTile = 0xffffffffu;
static_assert(kBlkTab <= 64, "pass block masks are 64-bit");
static_assert(kPassBlk >= 6, "one tile reads up to six blocks");
static_assert(kRingRows % (kThreads / (kSlab / 4)) == 0, "staging sweeps cover the ring");

// tile descriptor: node-relative slots
//   [0,7) ra   first row slot        [7,14) ca   first slot of column block A
//   [14,21) cb first slot of column block B      [21] column block B present
//   [22,24) kind (0 F, 1 U, 2 U2)    [24,27) node index in the batch
constexpr uint32_t kKindF = 0, kKindU = 1, kKindU2 = 2;
__device__ __forceinline__ uint32_t make_tile(uint32_t v, uint32_t kind, uint32_t ra, uint32_t ca,
                                              uint32_t cb, bool has_b) {
    return ra | (ca << 7) | ((cb & 127u) << 14) | (uint32_t(has_b) << 21) | (kind << 22) |
           (v << 24);
}

struct Geom5 {
    uint32_t nn, no, fn, fo, m;
    __device__ __forceinline__ void set(uint32_t nn_, uint32_t no_) {
        nn = nn_;
        no = no_;
        fn = nn - nn % 5;
        fo = no - no % 5;
        m = nn + no;
    }
    __device__ __forceinline__ uint32_t f_tiles() const {
        const uint32_t nfb = fn / 5, nob = fo / 5;
        uint32_t t = 0;
        for (uint32_t i = 0; i < nfb; ++i) t += (nfb - i + nob + 1) / 2;
        return t;
    }
    __device__ __forceinline__ uint32_t u_tiles() const { return nn > fn ? (m + 9) / 10 : 0u; }
    __device__ __forceinline__ uint32_t u2_tiles() const {
        return (no > fo && fn) ? (fn + 9) / 10 : 0u;
    }
    // t-th fused tile
    __device__ __forceinline__ uint32_t f_tile(uint32_t v, uint32_t t) const {
        const uint32_t nfb = fn / 5, nob = fo / 5;
        uint32_t i = 0;
        while (t >= (nfb - i + nob + 1) / 2) {
            t -= (nfb - i + nob + 1) / 2;
            ++i;
        }
        const uint32_t len = nfb - i + nob, q0 = 2 * t, q1 = 2 * t + 1;
        auto col = [&](uint32_t q) { return q < nfb - i ? 5 * (i + q) : nn + 5 * (q - (nfb - i)); };
        return make_tile(v, kKindF, 5 * i, col(q0), q1 < len ? col(q1) : 0u, q1 < len);
    }
    // t-th unfused tile (U tiles first, then U2)
    __device__ __forceinline__ uint32_t u_tile(uint32_t v, uint32_t t) const {
        const uint32_t nu = u_tiles();
        if (t < nu) return make_tile(v, kKindU, fn, 10 * t, 10 * t + 5, 10 * t + 5 < m);
        t -= nu;
        return make_tile(v, kKindU2, nn + fo, 10 * t, 10 * t + 5, 10 * t + 5 < fn);
    }
};

struct Shared5 {
    // the slab ring follows this struct in dynamic shared memory
    uint32_t colrow[kSlotTab];   // batch slot -> data row id (~0: none)
    float colmax[kSlotTab];      // batch slot -> candidate's row maximum
    uint32_t rowcnt[kSlotTab];   // proposals kept per candidate row
    uint32_t tiles[kMaxTiles];
    uint8_t blkpos[kBlkTab];     // pass mode: batch 8-slot block -> ring position
    uint8_t blklist[kPassBlk + 2];
    uint32_t ringrow[kRingRows];  // pass mode: ring row -> data row (~0: none)
    uint32_t n_tiles, pass_len, slot_budget, qn;
    uint4 q[2 * kMaxBatch];      // claimed-but-unbatched active-node records
    struct Batch {
        uint32_t node[kMaxBatch], vnn[kMaxBatch], vno[kMaxBatch], colbase[kMaxBatch];
        unsigned long long doff[kMaxBatch];
        uint32_t nv, nslots;
    } bd[2];
};

__device__ __forceinline__ void cp_async16(float* smem_dst, const float* gmem_src) {
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <uint32_t kPending>
__device__ __forceinline__ void cp_async_wait_pending() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kPending));
}

constexpr size_t kRingOffset = (sizeof(Shared5) + 127) / 128 * 128;
// eight spare rows: a tile's last rows may overhang its node (masked pairs)
constexpr size_t kSmem5 = kRingOffset + size_t(kStages * kRingRows + 8) * kPitch * sizeof(float);
static_assert(kSmem5 + 1024 <= 228 * 1024 / 4, "four CTAs per SM");

__device__ __forceinline__ float* ring5(Shared5& sh) {
    return reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(&sh) + kRingOffset);
}

// One 32-float slab of a 5 x 10 tile.  pa / pb / pc: element l8 of the tile's
// first row and of the first rows of its two column blocks; rows are kPitch
// apart.  acc[5 x + j] holds pairs (x, 2j) and (x, 2j + 1), columns 0..4 in
// block A and 5..9 in block B.  Arithmetic as join.cu's tile_slab: diff =
// fma(b, -1, a) == a - b, then fma(diff, diff, acc) on fused tiles or
// acc + fma(diff, diff, -0) (the rounded square; -0 opaque to ptxas) on
// unfused ones.
template <bool kFusedTile>
__device__ __forceinline__ void slab5(const float* __restrict__ pa, const float* __restrict__ pb,
                                      const float* __restrict__ pc, uint32_t nseg,
                                      float2 minus_zero, float2 (&acc)[25]) {
    const float2 minus_one = make_float2(-1.0f, -1.0f);
#pragma unroll
    for (uint32_t s = 0; s < kSlab / 8; ++s) {
        if (s >= nseg) break;  // the row's last slab may be partial (stride % 32)
        float a[5];
        float2 b[5];
#pragma unroll
        for (uint32_t x = 0; x < 5; ++x) a[x] = pa[x * kPitch + 8 * s];
        b[0] = make_float2(pb[0 * kPitch + 8 * s], pb[1 * kPitch + 8 * s]);
        b[1] = make_float2(pb[2 * kPitch + 8 * s], pb[3 * kPitch + 8 * s]);
        b[2] = make_float2(pb[4 * kPitch + 8 * s], pc[0 * kPitch + 8 * s]);
        b[3] = make_float2(pc[1 * kPitch + 8 * s], pc[2 * kPitch + 8 * s]);
        b[4] = make_float2(pc[3 * kPitch + 8 * s], pc[4 * kPitch + 8 * s]);
#pragma unroll
        for (uint32_t x = 0; x < 5; ++x) {
            const float2 ax = make_float2(a[x], a[x]);
#pragma unroll
            for (uint32_t j = 0; j < 5; ++j) {
                const float2 diff = __ffma2_rn(b[j], minus_one, ax);
                if (kFusedTile) {
                    acc[5 * x + j] = __ffma2_rn(diff, diff, acc[5 * x + j]);
                } else {
                    const float2 sq = __ffma2_rn(diff, diff, minus_zero);
                    acc[5 * x + j] = __fadd2_rn(acc[5 * x + j], sq);
                }
            }
        }
    }
}

__device__ __forceinline__ float acc5_at(const float2 (&acc)[25], uint32_t p) {
    if (p >= 50) return 0.0f;
    return (p & 1u) ? acc[p >> 1].y : acc[p >> 1].x;
}

// Reduce-scatter of the 50 per-lane partial sums (padded to 56) over the
// group's 8 lanes in the reference's tree order ((0+1)+(2+3))+((4+5)+(6+7))
// (distance.hpp:29-51).  Lane l8 = b0 + 2 b1 + 4 b2 ends with the sums of
// pairs [28 b0 + 14 b1 + 7 b2, + 7).
__device__ __forceinline__ void group_reduce56(const float2 (&acc)[25], uint32_t l8,
                                               float (&out)[7]) {
    const bool b0 = l8 & 1u, b1 = (l8 >> 1) & 1u, b2 = (l8 >> 2) & 1u;
    float r28[28];
#pragma unroll
    for (uint32_t j = 0; j < 28; ++j) {
        const float lo = acc5_at(acc, j), hi = acc5_at(acc, 28 + j);
        const float send = b0 ? lo : hi, keep = b0 ? hi : lo;
        r28[j] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 1));
    }
    float r14[14];
#pragma unroll
    for (uint32_t j = 0; j < 14; ++j) {
        const float send = b1 ? r28[j] : r28[14 + j], keep = b1 ? r28[14 + j] : r28[j];
        r14[j] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 2));
    }
#pragma unroll
    for (uint32_t j = 0; j < 7; ++j) {
        const float send = b2 ? r14[j] : r14[7 + j], keep = b2 ? r14[7 + j] : r14[j];
        out[j] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 4));
    }
}

__global__ void __launch_bounds__(kThreads, 4) join5_kernel(GraphView g, CandView c,
                                                            IterCounters* ctr,
                                                            uint32_t res_slots,
                                                            float minus_zero) {
    const float2 mz2 = make_float2(minus_zero, minus_zero);  // -0.0f, opaque to ptxas
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Shared5& sh = *reinterpret_cast<Shared5*>(smem_raw);
    const uint32_t tid = threadIdx.x, group = tid >> 3, l8 = tid & 7u;
    const uint32_t stride = g.stride, cap = c.cap;
    if (ctr->overflow || ctr->halt) return;
    const uint32_t n_active = ctr->active;
    const uint32_t n_slabs = (stride + kSlab - 1) / kSlab;
    const bool resident = res_slots != 0;
    if (tid == 0) {
        sh.qn = 0;
        sh.slot_budget = resident ? res_slots : kSlotTab;
    }
    if (tid < kBlkTab) sh.blkpos[tid] = 0;
    uint32_t gslab = 0;  // pass mode: slabs staged so far (ring stage = gslab % kStages)
    uint32_t a_next = 0;
    if (tid == 0) a_next = atomicAdd(&ctr->work, kMaxBatch);

    // warp 0 forms a batch (as join.cu): top the queue up with the claimed
    // chunk, claim the next, take the longest prefix whose slots and tiles fit
    auto form_batch = [&](Shared5::Batch& D) {
        const uint32_t lane = tid;
        uint32_t qn = sh.qn;
        const uint32_t a = __shfl_sync(0xffffffffu, a_next, 0);
        if (qn < kMaxBatch && a < n_active) {
            if (lane < kMaxBatch && a + lane < n_active) sh.q[qn + lane] = c.arec[a + lane];
            qn += min(kMaxBatch, n_active - a);
            if (lane == 0) a_next = atomicAdd(&ctr->work, kMaxBatch);
            __syncwarp();
        }
        uint32_t s_l = 0, t_l = 0, u = 0, nn = 0, no = 0;
        uint4 rec = make_uint4(0, 0, 0, 0);
        if (lane < qn) {
            rec = sh.q[lane];
            u = rec.x;
            nn = rec.y & 0xffffu;
            no = rec.y >> 16;
            Geom5 ng;
            ng.set(nn, no);
            s_l = ng.m;
            t_l = ng.f_tiles() + ng.u_tiles() + ng.u2_tiles();
        }
        uint32_t si = s_l, ti = t_l;
#pragma unroll
        for (uint32_t o = 1; o < 32; o <<= 1) {
            const uint32_t sp = __shfl_up_sync(0xffffffffu, si, o);
            const uint32_t tp = __shfl_up_sync(0xffffffffu, ti, o);
            if (lane >= o) {
                si += sp;
                ti += tp;
            }
        }
        const bool fit = lane < qn && lane < kMaxBatch &&
                         (lane == 0 || (si <= sh.slot_budget && ti <= kMaxTiles - 8));
        const uint32_t nv = __popc(__ballot_sync(0xffffffffu, fit));  // a prefix
        __syncwarp();
        if (lane < nv) {
            D.node[lane] = u;
            D.vnn[lane] = nn;
            D.vno[lane] = no;
            D.colbase[lane] = si - s_l;
            D.doff[lane] = uint64_t(rec.z) | (uint64_t(rec.w) << 32);
        } else if (lane < qn) {
            sh.q[lane - nv] = rec;
        }
        if (nv > 0 && lane == nv - 1) D.nslots = si;
        if (lane == 0) {
            sh.qn = qn - nv;
            D.nv = nv;
            if (nv == 0) D.nslots = 0;
        }
    };
    // slot contents (candidate id, row maximum) of batch D, loaded into
    // registers one batch ahead
    constexpr uint32_t kSlotsPerThread = (kSlotTab + kThreads - 1) / kThreads;
    uint32_t pf_id[kSlotsPerThread];
    float pf_max[kSlotsPerThread];
    auto load_slots = [&](const Shared5::Batch& D) {
#pragma unroll
        for (uint32_t j = 0; j < kSlotsPerThread; ++j) {
            const uint32_t sidx = tid + kThreads * j;
            pf_id[j] = 0xffffffffu;
            pf_max[j] = 0.0f;
            if (D.nv > 0 && sidx < D.nslots) {
                uint32_t v = 0;
                while (v + 1 < D.nv && D.colbase[v + 1] <= sidx) ++v;
                const uint32_t x = sidx - D.colbase[v], nn = D.vnn[v];
                const uint32_t pos = x < nn ? x : cap + x - nn;
                const size_t base = size_t(D.node[v]) * 2 * cap;
                pf_id[j] = c.ids[base + pos];
                pf_max[j] = c.filter ? c.cmax[base + pos] : __int_as_float(0x7f800000);
            }
        }
    };

    uint32_t cur = 0;
    __syncthreads();
    if (tid < 32) form_batch(sh.bd[0]);
    __syncthreads();
    load_slots(sh.bd[0]);
    while (true) {
        const Shared5::Batch& B = sh.bd[cur];
        const uint32_t nv = B.nv;
        if (nv == 0) break;
        const uint32_t nslots = B.nslots;
#pragma unroll
        for (uint32_t j = 0; j < kSlotsPerThread; ++j) {
            const uint32_t sidx = tid + kThreads * j;
            if (sidx < ((nslots + 7u) & ~7u)) {  // the last block's tail reads as "no row"
                sh.colrow[sidx] = pf_id[j];
                sh.colmax[sidx] = pf_max[j];
                sh.rowcnt[sidx] = 0;
            }
        }
        if (tid < 32) form_batch(sh.bd[cur ^ 1u]);
        __syncthreads();
        load_slots(sh.bd[cur ^ 1u]);  // consumed by the next iteration
        if (resident) {
            // the batch's rows, all slabs, staged once: slab s of slot r at
            // ring row s * res_slots + r
            constexpr uint32_t kC4 = kSlab / 4;
            const uint32_t j = tid % kC4;
            float* ring = ring5(sh);
            for (uint32_t s = 0; s < n_slabs; ++s) {
                const uint32_t e = s * kSlab + 4 * j;
                if (e >= stride) continue;
                for (uint32_t slot = tid / kC4; slot < nslots; slot += kThreads / kC4) {
                    const uint32_t row = sh.colrow[slot];
                    cp_async16(ring + size_t(s * res_slots + slot) * kPitch + 4 * j,
                               g.data + size_t(row) * stride + e);
                }
            }
            cp_async_commit();
        }
        // the batch's tiles: every node's fused tiles, padding to a whole
        // warp, then the unfused ones, so each warp runs one path
        if (tid < 32) {
            const uint32_t lane = tid;
            uint32_t cf_l = 0, cu_l = 0;
            if (lane < nv) {
                Geom5 ng;
                ng.set(B.vnn[lane], B.vno[lane]);
                cf_l = ng.f_tiles();
                cu_l = ng.u_tiles() + ng.u2_tiles();
            }
            uint32_t nt = 0;
            for (uint32_t phase = 0; phase < 2; ++phase) {
                const uint32_t mine = phase ? cu_l : cf_l;
                uint32_t incl = mine;
#pragma unroll
                for (uint32_t o = 1; o < kMaxBatch; o <<= 1) {
                    const uint32_t p = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += p;
                }
                const uint32_t total = __shfl_sync(0xffffffffu, incl, kMaxBatch - 1);
                for (uint32_t t0 = 0; t0 < total; t0 += 32) {
                    const uint32_t t = t0 + lane;
                    // node v: the first with incl[v] > t
                    uint32_t v = 0, before = 0;
                    for (uint32_t w = 0; w < kMaxBatch; ++w) {
                        const uint32_t iw = __shfl_sync(0xffffffffu, incl, w);
                        if (iw <= t) {
                            v = w + 1;
                            before = iw;
                        }
                    }
                    if (t < total) {
                        Geom5 ng;
                        ng.set(B.vnn[v], B.vno[v]);
                        sh.tiles[nt + t] = phase ? ng.u_tile(v, t - before) : ng.f_tile(v, t - before);
                    }
                }
                nt += total;
                if (phase == 0) {  // pad the fused run to whole warps
                    const uint32_t padded = (nt + 3u) & ~3u;
                    if (lane < padded - nt) sh.tiles[nt + lane] = kDeadTile;
                    nt = padded;
                }
            }
            if (lane == 0) sh.n_tiles = nt;
        }
        if (resident) cp_async_wait_pending<0>();
        __syncthreads();
        const uint32_t n_tiles = sh.n_tiles;

        uint32_t pass_len = kGroups;
        for (uint32_t t0 = 0; t0 < n_tiles; t0 += pass_len) {
            if (!resident) {
                // warp 0 schedules the pass: the longest run of whole warps'
                // tiles (<= 16) whose 8-slot blocks fit kPassBlk ring positions
                if (tid < 32) {
                    const uint32_t lane = tid, left = min(kGroups, n_tiles - t0);
                    uint64_t m = 0;
                    if (lane < left) {
                        const uint32_t tile = sh.tiles[t0 + lane];
                        if (tile != kDeadTile) {
                            const uint32_t v = tile >> 24, kind = (tile >> 22) & 3u;
                            const uint32_t ra = tile & 127u, ca = (tile >> 7) & 127u,
                                           cb = (tile >> 14) & 127u;
                            Geom5 ng;
                            ng.set(B.vnn[v], B.vno[v]);
                            const uint32_t base = B.colbase[v];
                            const uint32_t rend = kind == kKindF ? ra + 5 : (kind == kKindU ? ng.nn : ng.m);
                            const uint32_t cend = kind == kKindF ? 128u : (kind == kKindU ? ng.m : ng.fn);
                            auto range = [&](uint32_t s0, uint32_t end) {
                                const uint32_t s1 = min(s0 + 5, end) - 1;  // last needed slot
                                return (1ull << ((base + s0) >> 3)) | (1ull << ((base + s1) >> 3));
                            };
                            m = range(ra, rend) | range(ca, cend);
                            if ((tile >> 21) & 1u) m |= range(cb, cend);
                        }
                    }
#pragma unroll
                    for (uint32_t o = 1; o < 32; o <<= 1) {
                        const uint64_t mp = __shfl_up_sync(0xffffffffu, m, o);
                        if (lane >= o) m |= mp;
                    }
                    // whole warps when the first four tiles fit (the usual
                    // case: a warp's tiles share rows); else as many as fit
                    const bool fits = lane < left && __popcll(m) <= kPassBlk;
                    const uint32_t fitm = __ballot_sync(0xffffffffu, fits);
                    const uint32_t okm = __ballot_sync(
                        0xffffffffu, fits && ((lane & 3u) == 3u || lane + 1 == left));
                    const uint32_t last = 31u - __clz(okm ? okm : fitm);
                    const uint64_t pm = __shfl_sync(0xffffffffu, m, last);
                    for (uint32_t bit = lane; bit < kBlkTab; bit += 32)
                        if ((pm >> bit) & 1ull) {
                            const uint32_t pos = __popcll(pm & ((1ull << bit) - 1ull));
                            sh.blkpos[bit] = uint8_t(pos);
                            sh.blklist[pos] = uint8_t(bit);
                        }
                    __syncwarp();
                    const uint32_t nrows = __popcll(pm) * 8u;
                    for (uint32_t r = lane; r < kRingRows; r += 32)
                        sh.ringrow[r] =
                            r < nrows ? sh.colrow[sh.blklist[r >> 3] * 8u + (r & 7u)] : 0xffffffffu;
                    if (lane == 0) sh.pass_len = last + 1;
                }
                __syncthreads();
                pass_len = sh.pass_len;
            }
            const uint32_t t = t0 + group;
            const uint32_t tile0 = group < pass_len && t < n_tiles ? sh.tiles[t] : kDeadTile;
            const bool live = tile0 != kDeadTile;
            const uint32_t tile = live ? tile0 : 0u;
            const uint32_t v = tile >> 24, kind = (tile >> 22) & 3u;
            const uint32_t ra = tile & 127u, ca = (tile >> 7) & 127u;
            const bool has_b = (tile >> 21) & 1u;
            const uint32_t cb = has_b ? (tile >> 14) & 127u : ca;
            const uint32_t base = B.colbase[v];
            float2 acc[25];
#pragma unroll
            for (uint32_t p = 0; p < 25; ++p) acc[p] = make_float2(0.0f, 0.0f);
            if (resident) {
                if (live) {
                    const float* pa = ring5(sh) + size_t(base + ra) * kPitch + l8;
                    const float* pb = ring5(sh) + size_t(base + ca) * kPitch + l8;
                    const float* pc = ring5(sh) + size_t(base + cb) * kPitch + l8;
                    const uint32_t slab_floats = res_slots * kPitch;
                    for (uint32_t s = 0; s < n_slabs; ++s) {
                        const uint32_t nseg = min(kSlab, stride - s * kSlab) / 8u;
                        if (kind == kKindF)
                            slab5<true>(pa, pb, pc, nseg, mz2, acc);
                        else
                            slab5<false>(pa, pb, pc, nseg, mz2, acc);
                        pa += slab_floats;
                        pb += slab_floats;
                        pc += slab_floats;
                    }
                }
            } else {
                auto ringpos = [&](uint32_t slot) {
                    return uint32_t(sh.blkpos[slot >> 3]) * 8u + (slot & 7u);
                };
                const uint32_t oa = live ? ringpos(base + ra) * kPitch + l8 : 0u;
                const uint32_t ob = live ? ringpos(base + ca) * kPitch + l8 : 0u;
                const uint32_t oc = live ? ringpos(base + cb) * kPitch + l8 : 0u;
                // kStages-deep cp.async ring, one barrier per slab; thread tid
                // stages 16-byte chunk tid % 8 of ring rows tid / 8 + 16 q
                constexpr uint32_t kC4 = kSlab / 4, kSweep = kThreads / kC4;
                constexpr uint32_t kRowsPerThread = kRingRows / kSweep;
                const uint32_t j = tid % kC4, r0 = tid / kC4;
                uint32_t my_rows[kRowsPerThread];
#pragma unroll
                for (uint32_t q = 0; q < kRowsPerThread; ++q) my_rows[q] = sh.ringrow[r0 + kSweep * q];
                float* const my_dst = ring5(sh) + r0 * kPitch + 4 * j;
                auto issue = [&](uint32_t sl) {
                    const uint32_t st = (gslab + sl) % kStages, e = sl * kSlab + 4 * j;
                    if (e < stride) {
                        float* const dst = my_dst + size_t(st) * kRingRows * kPitch;
#pragma unroll
                        for (uint32_t q = 0; q < kRowsPerThread; ++q)
                            if (my_rows[q] != 0xffffffffu)
                                cp_async16(dst + q * kSweep * kPitch,
                                           g.data + size_t(my_rows[q]) * stride + e);
                    }
                    cp_async_commit();
                };
                for (uint32_t p = 0; p < kStages - 1; ++p) {
                    if (p < n_slabs)
                        issue(p);
                    else
                        cp_async_commit();
                }
                for (uint32_t sl = 0; sl < n_slabs; ++sl) {
                    const uint32_t st = (gslab + sl) % kStages;
                    cp_async_wait_pending<kStages - 2>();  // slab sl has landed
                    __syncthreads();  // for every thread; and slab sl - 1's stage is free
                    if (sl + kStages - 1 < n_slabs)
                        issue(sl + kStages - 1);
                    else
                        cp_async_commit();
                    const float* stage = ring5(sh) + size_t(st) * kRingRows * kPitch;
                    const uint32_t nseg = min(kSlab, stride - sl * kSlab) / 8u;
                    if (live) {
                        if (kind == kKindF)
                            slab5<true>(stage + oa, stage + ob, stage + oc, nseg, mz2, acc);
                        else
                            slab5<false>(stage + oa, stage + ob, stage + oc, nseg, mz2, acc);
                    }
                }
                gslab += n_slabs;
            }
            float sums[7];
            group_reduce56(acc, l8, sums);
            if (live) {
                Geom5 ng;
                ng.set(B.vnn[v], B.vno[v]);
                const uint32_t nn = ng.nn, m = ng.m, fn = ng.fn;
                uint64_t* const D = c.D + B.doff[v];
                const uint32_t p0 = 28u * (l8 & 1u) + 14u * ((l8 >> 1) & 1u) + 7u * ((l8 >> 2) & 1u);
#pragma unroll
                for (uint32_t q = 0; q < 7; ++q) {
                    const uint32_t p = p0 + q;
                    if (p >= 50) break;
                    const uint32_t x = p / 10u, y = p % 10u;
                    if (y >= 5 && !has_b) continue;
                    const uint32_t r = ra + x, cc = y < 5 ? ca + y : cb + (y - 5);
                    // every evaluated pair exactly once, in the reference's class
                    bool ok;
                    if (kind == kKindF)
                        ok = cc >= nn || cc > r;  // r < fn; new block j >= i, or a full old block
                    else if (kind == kKindU)
                        ok = r < nn && cc < m && (cc >= nn || cc < fn || cc > r);
                    else
                        ok = r < m && cc < fn;
                    if (!ok) continue;
                    const uint32_t sr = base + r, sc = base + cc;
                    const uint32_t id_r = sh.colrow[sr], id_c = sh.colrow[sc];
                    // an id listed twice pairs with itself: try_insert ignores
                    // self (graph.hpp:116-129)
                    if (c.filter && id_r == id_c) continue;
                    const float dist = sums[q];
                    if (dist < sh.colmax[sr]) {
                        const uint32_t pos = atomicAdd(&sh.rowcnt[sr], 1u);
                        D[prow(r, nn, m) + 1 + pos] = pack_key(dist, id_c);
                    }
                    if (dist < sh.colmax[sc]) {
                        const uint32_t pos = atomicAdd(&sh.rowcnt[sc], 1u);
                        D[prow(cc, nn, m) + 1 + pos] = pack_key(dist, id_r);
                    }
                }
            }
        }
        // row counts of the batch's proposal blocks
        __syncthreads();
        for (uint32_t v = 0; v < nv; ++v) {
            const uint32_t nn = B.vnn[v], m = nn + B.vno[v];
            for (uint32_t r = tid; r < m; r += kThreads)
                c.D[B.doff[v] + prow(r, nn, m)] = sh.rowcnt[B.colbase[v] + r];
        }
        __syncthreads();  // the next batch rewrites the slot tables
        cur ^= 1u;
    }
}

}  // namespace

void launch_join5(const GraphView& g, const CandView& c, IterCounters* ctr, uint32_t max_active,
                  cudaStream_t s) {
    if (!max_active) return;
    // resident mode when every slab of a batch's rows fits the ring with a
    // slot budget of at least one full node (2 cap slots); otherwise pass mode
    const uint32_t n_slabs = (g.stride + kSlab - 1) / kSlab;
    uint32_t res_slots = std::min<uint32_t>(kSlotTab, kStages * kRingRows / n_slabs / 8 * 8);
    static const bool allow_resident = [] {
        const char* v = getenv("KNNG_JOIN_RESIDENT");
        return !(v && v[0] == '0');
    }();
    if (res_slots < 2 * c.cap || !allow_resident) res_slots = 0;
    static int occ[kMaxDevices] = {};  // per device: the attribute is per device
    int& per_sm = occ[current_device()];
    if (!per_sm) {
        check_launch(cudaFuncSetAttribute(join5_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(kSmem5)));
        int v = 0;
        check_launch(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, join5_kernel, int(kThreads),
                                                                   kSmem5));
        per_sm = v < 1 ? 1 : v;
    }
    uint32_t grid = device_sm_count() * uint32_t(per_sm);
    if (grid > max_active) grid = max_active;
    check_launch(cudaMemsetAsync(&ctr->work, 0, sizeof(uint32_t), s));
    join5_kernel<<<grid, kThreads, kSmem5, s>>>(g, c, ctr, res_slots, -0.0f);
}

}  // namespace knng_cuda
