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
// tile boundaries.  A node's candidates take slots in the order
//   [ fn fused new | r = nn % 5 leftover new | ro = no % 5 leftover old | fo fused old ]
// (no padding inside a node or between the nodes of a batch), and its pairs
// run as
//   F (fused)    new rows [5i, 5i + 5) x two 5-blocks out of
//                {new blocks j >= i (j == i: the triangle)} ++ {full old blocks}
//   U (unfused)  the leftover rows -- the r leftover new candidates against
//                every column, and (when the node has fused new candidates) the
//                ro leftover old candidates against the fused new ones -- share
//                the row block [fn, fn + 5): 5 x 10 tiles over the columns; a
//                second row block only when r + ro > 5
//   T (unfused)  the same leftover rows when r + ro <= 2: thin 2 x 24 tiles
//                (a late node with one new and 23 old candidates is one tile of
//                48 pair slots instead of three of 50)
// nn = 7, no = 23: 3 F + 3 U tiles of 50 pairs against ten 8 x 8 tiles.
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

#include "join5_geom.cuh"
#include "kernels.cuh"
#include "tile_math.cuh"

namespace knng_cuda {

namespace {

#ifndef KNNG_T5_CHECKS
#define KNNG_T5_CHECKS 0  // 1: device-side bounds checks with a message (diagnostics build)
#endif
#if KNNG_T5_CHECKS
#define T5CHECK(cond, what, a, b)                                                        \
    do {                                                                                \
        if (!(cond)) {                                                                  \
            printf("join5 check failed: %s (%u, %u) block %d thread %d\n", what,       \
                   unsigned(a), unsigned(b), int(blockIdx.x), int(threadIdx.x));      \
            __trap();                                                                   \
        }                                                                               \
    } while (0)
#else
#define T5CHECK(cond, what, a, b) ((void)0)
#endif

#ifndef KNNG_T5_THREADS
#define KNNG_T5_THREADS 128
#endif
constexpr uint32_t kThreads = KNNG_T5_THREADS;  // 16 groups of 8 lanes
constexpr uint32_t kGroups = kThreads / 8;
#ifndef KNNG_T5_SLAB
#define KNNG_T5_SLAB 32
#endif
#ifndef KNNG_T5_STAGES
#define KNNG_T5_STAGES 3
#endif
constexpr uint32_t kSlab = KNNG_T5_SLAB;      // floats per row per ring stage
constexpr uint32_t kStages = KNNG_T5_STAGES;
// Ring rows are kPitch floats apart: 36 puts rows r and r + 10 (the column
// blocks of the four tiles a warp usually runs) 8 banks apart, and rows r and
// r + 5 20 banks apart, so the groups' 8-bank reads do not collide.
constexpr uint32_t kPitch = kSlab + 4;
#ifndef KNNG_T5_PASSBLK
#define KNNG_T5_PASSBLK 14
#endif
constexpr uint32_t kPassBlk = KNNG_T5_PASSBLK;  // 8-slot blocks one pass may stage
constexpr uint32_t kRingRows = kPassBlk * 8;
#ifndef KNNG_T5_MAXBATCH
#define KNNG_T5_MAXBATCH 8
#endif
constexpr uint32_t kMaxBatch = KNNG_T5_MAXBATCH;  // nodes per batch (tile descriptors hold 4 bits)
static_assert(kMaxBatch <= 16, "node index field of a tile descriptor");
#ifndef KNNG_T5_SLOTTAB
#define KNNG_T5_SLOTTAB 320
#endif
constexpr uint32_t kSlotTab = KNNG_T5_SLOTTAB;  // batch slots
constexpr uint32_t kBlkTab = kSlotTab / 8;
#ifndef KNNG_T5_MAXTILES
#define KNNG_T5_MAXTILES 384
#endif
constexpr uint32_t kMaxTiles = KNNG_T5_MAXTILES;
constexpr uint32_t kDeadTile = 3u << 22;   // kind 3: padding, no work
constexpr uint32_t kGroupEnd = 1u << 28;   // last tile of a pass group

#ifndef KNNG_T5_ENDMIN
#define KNNG_T5_ENDMIN 17  // off: measured no gain (C5 391 vs 388 ms with 12 vs off)
#endif
constexpr uint32_t kEndMin = KNNG_T5_ENDMIN;  // fewest tiles of a pass cut short at a group boundary
constexpr uint32_t kGroupSlots = (kPassBlk - 1) * 8;  // a pass group's slots fit one pass
static_assert(kBlkTab <= 64, "pass block masks are 64-bit");
static_assert(kPassBlk >= 6, "one tile reads up to six blocks");
static_assert(kRingRows % (kThreads / (kSlab / 4)) == 0, "staging sweeps cover the ring");

// (tile descriptors and Geom5: join5_geom.cuh)
using namespace t5;
#ifndef KNNG_T5_THIN
#define KNNG_T5_THIN 1
#endif

struct Shared5 {
    // the slab ring follows this struct in dynamic shared memory
    uint32_t colrow[kSlotTab];   // batch slot -> data row id (~0: none)
    float colmax[kSlotTab];      // batch slot -> candidate's row maximum
    uint32_t rowcnt[kSlotTab];   // per candidate row: write cursor in the node's proposal block
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

// Dynamic shared memory: the slab ring first, then the tables.  A tile's last
// rows may overhang its node and a thin tile reads 24 consecutive ring rows
// whatever its live width, so reads can run up to 23 rows past the ring's end:
// they land in the tables (masked pairs, any bit pattern will do).
constexpr size_t kRingBytes = size_t(kStages) * kRingRows * kPitch * sizeof(float);
constexpr size_t kSmem5 = kRingBytes + sizeof(Shared5);
static_assert(kRingBytes % 16 == 0, "tables stay 16-byte aligned");
static_assert(sizeof(Shared5) >= (kThinCols - 1) * kPitch * sizeof(float), "overhang stays inside");
#ifndef KNNG_T5_CTAS
#define KNNG_T5_CTAS 4
#endif
static_assert(kSmem5 + 1024 <= 228 * 1024 / KNNG_T5_CTAS, "CTAs per SM");

__device__ __forceinline__ float* ring5(Shared5& sh) {
    return reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(&sh) - kRingBytes);
}

// One 32-float slab of a 5 x 10 tile.  pa / pb / pc: element l8 of the tile's
// first row and of the first rows of its two column blocks; rows are kPitch
// apart.  acc[5 x + j] holds pairs (x, 2j) and (x, 2j + 1), columns 0..4 in
// block A and 5..9 in block B.  Arithmetic as join.cu's tile_slab: diff =
// fma(b, -1, a) == a - b, then fma(diff, diff, acc) on fused tiles or
// acc + fma(diff, diff, -0) (the rounded square; -0 opaque to ptxas) on
// unfused ones.
// (seg5: one 8-float segment.  A slab without the per-segment exit test lets
// ptxas hoist loads across segments but costs spills: C5 -0.4%, C4 +5%.)
template <bool kFusedTile>
__device__ __forceinline__ void seg5(const float* __restrict__ pa, const float* __restrict__ pb,
                                     const float* __restrict__ pc, uint32_t s, float2 minus_zero,
                                     float2 (&acc)[25]) {
    const float2 minus_one = make_float2(-1.0f, -1.0f);
    {
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
template <bool kFusedTile>
__device__ __forceinline__ void slab5(const float* __restrict__ pa, const float* __restrict__ pb,
                                      const float* __restrict__ pc, uint32_t nseg,
                                      float2 minus_zero, float2 (&acc)[25]) {
#pragma unroll
    for (uint32_t s = 0; s < kSlab / 8; ++s) {
        if (s >= nseg) break;  // the row's last slab may be partial (stride % 32)
        seg5<kFusedTile>(pa, pb, pc, s, minus_zero, acc);
    }
}

// One 32-float slab of a thin 2 x 24 unfused tile.  pa: element l8 of the first
// of the two rows, pb: of the first of 24 consecutive column rows.
// acc[12 x + j] holds pairs (x, 2j) and (x, 2j + 1); acc[24] stays zero.
__device__ __forceinline__ void seg_thin(const float* __restrict__ pa,
                                         const float* __restrict__ pb, uint32_t s,
                                         float2 minus_zero, float2 (&acc)[25]) {
    const float2 minus_one = make_float2(-1.0f, -1.0f);
    {
        const float a0 = pa[8 * s], a1 = pa[kPitch + 8 * s];
        const float2 ax0 = make_float2(a0, a0), ax1 = make_float2(a1, a1);
#pragma unroll
        for (uint32_t j = 0; j < kThinCols / 2; ++j) {
            const float2 b = make_float2(pb[(2 * j) * kPitch + 8 * s], pb[(2 * j + 1) * kPitch + 8 * s]);
            const float2 d0 = __ffma2_rn(b, minus_one, ax0);
            const float2 d1 = __ffma2_rn(b, minus_one, ax1);
            acc[j] = __fadd2_rn(acc[j], __ffma2_rn(d0, d0, minus_zero));
            acc[kThinCols / 2 + j] = __fadd2_rn(acc[kThinCols / 2 + j], __ffma2_rn(d1, d1, minus_zero));
        }
    }
}
__device__ __forceinline__ void slab_thin(const float* __restrict__ pa,
                                          const float* __restrict__ pb, uint32_t nseg,
                                          float2 minus_zero, float2 (&acc)[25]) {
#pragma unroll
    for (uint32_t s = 0; s < kSlab / 8; ++s) {
        if (s >= nseg) break;
        seg_thin(pa, pb, s, minus_zero, acc);
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

// Three instantiations (a third of the code each: the short-row configs were
// stalling on instruction fetch with everything in one kernel):
//   kModeResident  short rows, a batch's rows staged once (C1, C4)
//   kModePass      rows streamed through the slab ring, a few slabs per pass
//                  (C3): per-pass set-up dominates, so the batch is one pass
//                  group (phase-major tile list, fewest passes) and there are
//                  no thin tiles
//   kModePassLong  rows of kLongRow floats or more (C5): node-major pass groups
//                  and thin tiles, which cut the rows staged per evaluation
constexpr int kModeResident = 0, kModePass = 1, kModePassLong = 2;
#ifndef KNNG_T5_LONGROW
#define KNNG_T5_LONGROW 512
#endif
constexpr uint32_t kLongRow = KNNG_T5_LONGROW;
template <int kMode>
__global__ void __launch_bounds__(kThreads, KNNG_T5_CTAS) join5_kernel(GraphView g, CandView c,
                                                                      IterCounters* ctr,
                                                                      uint32_t res_slots,
                                                                      float minus_zero) {
    constexpr bool kResident = kMode == kModeResident;
    constexpr bool kGrouped = kMode == kModePassLong;
    constexpr bool kThinOK = KNNG_T5_THIN && kMode == kModePassLong;
    const float2 mz2 = make_float2(minus_zero, minus_zero);  // -0.0f, opaque to ptxas
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Shared5& sh = *reinterpret_cast<Shared5*>(smem_raw + kRingBytes);
    const uint32_t tid = threadIdx.x, group = tid >> 3, l8 = tid & 7u;
    const uint32_t stride = g.stride, cap = c.cap;
    if (ctr->overflow || ctr->halt) return;
    const uint32_t n_active = ctr->active;
    const uint32_t n_slabs = (stride + kSlab - 1) / kSlab;
    constexpr bool resident = kResident;
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
            ng.set(nn, no, kThinOK);
            s_l = ng.m;
            t_l = ((ng.f_tiles() + 3u) & ~3u) + ((ng.u_tiles() + 3u) & ~3u) + ((ng.t_tiles() + 3u) & ~3u);
            if (t_l < kGroups) t_l = kGroups;  // an upper bound of its share of the tile list
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
                         (lane == 0 || (si <= sh.slot_budget && ti <= kMaxTiles));
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
                Geom5 ng;
                ng.set(nn, D.vno[v], kThinOK);
                const uint32_t pos = x < nn ? x : cap + ng.cand(x) - nn;
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
                // the row's write cursor: word index, in the node's proposal
                // block, of the next key (the row's first word is its count)
                uint32_t cursor = 0;
                if (sidx < nslots) {
                    uint32_t v = 0;
                    while (v + 1 < nv && B.colbase[v + 1] <= sidx) ++v;
                    Geom5 ng;
                    ng.set(B.vnn[v], B.vno[v], kThinOK);
                    cursor = uint32_t(prow(ng.cand(sidx - B.colbase[v]), ng.nn, ng.m)) + 1u;
                }
                sh.rowcnt[sidx] = cursor;
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
        // The batch's tiles.  Nodes are taken in pass groups: consecutive nodes
        // whose tiles fill at most one pass (16 tiles, kGroupSlots slots), so
        // that a node's rows are staged once for all of its tiles; a node with
        // more tiles is a group of its own.  Inside a group: the 5 x 10
        // leftover-row tiles of its nodes, the thin ones, then the fused ones
        // (a big node's later fused row blocks read only its later columns),
        // each run padded to a whole warp so that each warp runs one path.
        // Resident mode stages the batch once, and short rows want the fewest
        // passes: there the whole batch is one group.
        if (tid < 32) {
            const uint32_t lane = tid;
            uint32_t cnt_l[3] = {0, 0, 0}, s_l = 0;  // F, U, T tiles; slots
            if (lane < nv) {
                Geom5 ng;
                ng.set(B.vnn[lane], B.vno[lane], kThinOK);
                cnt_l[0] = ng.f_tiles();
                cnt_l[1] = ng.u_tiles();
                cnt_l[2] = ng.t_tiles();
                s_l = ng.m;
            }
            auto pad4 = [](uint32_t x) { return (x + 3u) & ~3u; };
            // every lane walks the nodes; lane v keeps node v's run offsets
            uint32_t gbase = 0, gfirst = 0, gf = 0, gu = 0, gt = 0, gs = 0;
            uint32_t pre[3] = {0, 0, 0}, off[3] = {0, 0, 0};
            uint32_t gend_l = 0;  // lane v: index of its group's last tile slot
            auto close = [&](uint32_t wend) {  // the group is nodes [gfirst, wend)
                const uint32_t pu = pad4(gu), pt = pad4(gt), pf = pad4(gf);
                uint32_t len = pu + pt + pf;
                if (lane >= gfirst && lane < wend) {
                    off[1] = gbase + pre[1];
                    off[2] = gbase + pu + pre[2];
                    off[0] = gbase + pu + pt + pre[0];
                    gend_l = gbase + len - 1;
                }
                gbase += len;
                gfirst = wend;
                gf = gu = gt = gs = 0;
            };
            for (uint32_t w = 0; w < nv; ++w) {
                const uint32_t fw = __shfl_sync(0xffffffffu, cnt_l[0], w);
                const uint32_t uw = __shfl_sync(0xffffffffu, cnt_l[1], w);
                const uint32_t tw = __shfl_sync(0xffffffffu, cnt_l[2], w);
                const uint32_t sw = __shfl_sync(0xffffffffu, s_l, w);
                if (kGrouped && w > gfirst &&
                    (pad4(gf + fw) + pad4(gu + uw) + pad4(gt + tw) > kGroups || gs + sw > kGroupSlots))
                    close(w);
                if (lane == w) {
                    pre[0] = gf;
                    pre[1] = gu;
                    pre[2] = gt;
                }
                gf += fw;
                gu += uw;
                gt += tw;
                gs += sw;
            }
            close(nv);
            const uint32_t nt = gbase;
            for (uint32_t t = lane; t < nt; t += 32) sh.tiles[t] = kDeadTile;
            __syncwarp();
#pragma unroll
            for (uint32_t phase = 0; phase < 3; ++phase) {
                uint32_t incl = cnt_l[phase];
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
                    const uint32_t ov = __shfl_sync(0xffffffffu, off[phase], v & 31u);
                    if (t < total) {
                        Geom5 ng;
                        ng.set(B.vnn[v], B.vno[v], kThinOK);
                        sh.tiles[ov + t - before] = phase == 0   ? ng.f_tile(v, t - before)
                                                    : phase == 1 ? ng.u_tile(v, t - before)
                                                                 : ng.t_tile(v, t - before);
                    }
                }
            }
            __syncwarp();
            if (lane < nv) atomicOr(&sh.tiles[gend_l], kGroupEnd);
            if (lane == 0) sh.n_tiles = nt;
            T5CHECK(nt <= kMaxTiles, "tile list", nt, kMaxTiles);
            T5CHECK(B.nslots <= sh.slot_budget || nv == 1, "batch slots", B.nslots, sh.slot_budget);
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
                        if (!tile_dead(tile)) {
                            const uint32_t v = (tile >> 24) & 15u, kind = (tile >> 22) & 3u;
                            const uint32_t ra = tile & 127u, ca = (tile >> 7) & 127u,
                                           cb = (tile >> 14) & 127u;
                            Geom5 ng;
                            ng.set(B.vnn[v], B.vno[v], kThinOK);
                            const uint32_t base = B.colbase[v];
                            // 8-slot blocks of the node's slots [s0, s1]
                            auto range = [&](uint32_t s0, uint32_t s1) {
                                const uint32_t lo = (base + s0) >> 3, hi = (base + s1) >> 3;
                                return ((2ull << hi) - 1ull) & ~((1ull << lo) - 1ull);
                            };
                            if (kind == kKindF) {
                                m = range(ra, ra + 4) | range(ca, ca + 4);
                                if ((tile >> 21) & 1u) m |= range(cb, cb + 4);
                            } else {
                                const uint32_t rend = ng.fn + ng.lrow, cend = ng.col_end(ra);
                                const uint32_t rows = kind == kKindU ? 5u : 2u;
                                m = range(ra, min(ra + rows, rend) - 1);
                                if (kind == kKindU) {
                                    m |= range(ca, min(ca + 5, cend) - 1);
                                    if ((tile >> 21) & 1u) m |= range(cb, min(cb + 5, cend) - 1);
                                } else {
                                    m |= range(ca, min(ca + kThinCols, cend) - 1);
                                }
                            }
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
                    // ... and end at a pass-group boundary when that still
                    // fills kEndMin groups: the next group then starts a pass
                    // and its rows are staged once
                    const uint32_t endm = __ballot_sync(
                        0xffffffffu, fits && (sh.tiles[t0 + min(lane, left - 1)] & kGroupEnd));
                    uint32_t pick = okm ? okm : fitm;
                    if ((endm & pick) >> (kEndMin - 1)) pick &= endm;
                    const uint32_t last = 31u - __clz(pick);
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
            const bool live = !tile_dead(tile0);
            const uint32_t tile = live ? tile0 : 0u;
            const uint32_t v = (tile >> 24) & 15u, kind = (tile >> 22) & 3u;
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
                        else if (kind == kKindU)
                            slab5<false>(pa, pb, pc, nseg, mz2, acc);
                        else
                            slab_thin(pa, pb, nseg, mz2, acc);
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
                T5CHECK(oa / kPitch + 5 <= kRingRows + 23 && ob / kPitch + (kind == kKindT ? kThinCols : 5) <= kRingRows + 23 &&
                            oc / kPitch + 5 <= kRingRows + 23,
                        "ring row", ob / kPitch, oc / kPitch);
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
                        else if (kind == kKindU)
                            slab5<false>(stage + oa, stage + ob, stage + oc, nseg, mz2, acc);
                        else
                            slab_thin(stage + oa, stage + ob, nseg, mz2, acc);
                    }
                }
                gslab += n_slabs;
            }
            float sums[7];
            group_reduce56(acc, l8, sums);
            if (live) {
                Geom5 ng;
                ng.set(B.vnn[v], B.vno[v], kThinOK);
                uint64_t* const D = c.D + B.doff[v];
                const uint32_t p0 = 28u * (l8 & 1u) + 14u * ((l8 >> 1) & 1u) + 7u * ((l8 >> 2) & 1u);
#pragma unroll
                for (uint32_t q = 0; q < 7; ++q) {
                    const uint32_t p = p0 + q;
                    if (p >= 50) break;
                    uint32_t r, cc;
                    if (!ng.tile_pair(tile, p, r, cc)) continue;
                    const uint32_t sr = base + r, sc = base + cc;
                    const uint32_t id_r = sh.colrow[sr], id_c = sh.colrow[sc];
                    // an id listed twice pairs with itself: try_insert ignores
                    // self (graph.hpp:116-129)
                    if (c.filter && id_r == id_c) continue;
                    const float dist = sums[q];
#if KNNG_T5_CHECKS
                    {
                        auto row_end = [&](uint32_t slot) {  // one past the row's last word
                            const uint32_t cd = ng.cand(slot);
                            return uint32_t(prow(cd, ng.nn, ng.m)) + (cd < ng.nn ? ng.m : ng.nn + 1u);
                        };
                        T5CHECK(r < ng.m && cc < ng.m && r != cc, "pair slots", r, cc);
                        T5CHECK(sh.rowcnt[sr] < row_end(r), "row cursor", sh.rowcnt[sr], row_end(r));
                        T5CHECK(sh.rowcnt[sc] < row_end(cc), "column cursor", sh.rowcnt[sc], row_end(cc));
                    }
#endif
                    if (dist < sh.colmax[sr]) D[atomicAdd(&sh.rowcnt[sr], 1u)] = pack_key(dist, id_c);
                    if (dist < sh.colmax[sc]) D[atomicAdd(&sh.rowcnt[sc], 1u)] = pack_key(dist, id_r);
                }
            }
        }
        // row counts of the batch's proposal blocks
        __syncthreads();
        for (uint32_t v = 0; v < nv; ++v) {
            Geom5 ng;
            ng.set(B.vnn[v], B.vno[v], kThinOK);
            for (uint32_t r = tid; r < ng.m; r += kThreads)
            {
                const uint32_t first = uint32_t(prow(ng.cand(r), ng.nn, ng.m));
                c.D[B.doff[v] + first] = sh.rowcnt[B.colbase[v] + r] - first - 1u;
            }
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
    // per device and instantiation: the attribute is per device
    static int occ[3][kMaxDevices] = {};
    const int mode = res_slots ? kModeResident : (g.stride >= kLongRow ? kModePassLong : kModePass);
    auto kernel = mode == kModeResident ? join5_kernel<kModeResident>
                  : mode == kModePass   ? join5_kernel<kModePass>
                                        : join5_kernel<kModePassLong>;
    int& per_sm = occ[mode][current_device()];
    if (!per_sm) {
        check_launch(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(kSmem5)));
        int v = 0;
        check_launch(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel, int(kThreads),
                                                                   kSmem5));
        per_sm = v < 1 ? 1 : v;
    }
    uint32_t grid = device_sm_count() * uint32_t(per_sm);
    if (grid > max_active) grid = max_active;
    check_launch(cudaMemsetAsync(&ctr->work, 0, sizeof(uint32_t), s));
    kernel<<<grid, kThreads, kSmem5, s>>>(g, c, ctr, res_slots, -0.0f);
}

}  // namespace knng_cuda

// Test hook (host only, no GPU): every pair the tiles of a node with nn new and
// no old candidates evaluate, as {row position, column position, fused} triples
// in candidate order (new list, then old list).  Returns the number of tiles;
// *count = the number of pairs (the first `capacity` are written).
extern "C" int knng_cuda_debug_join5_pairs(uint32_t nn, uint32_t no, int thin, uint32_t* out,
                                           uint32_t capacity, uint32_t* count) {
    using namespace knng_cuda::t5;
    Geom5 ng;
    ng.set(nn, no, thin != 0);
    uint32_t n_pairs = 0, n_tiles = 0;
    auto emit = [&](uint32_t tile) {
        ++n_tiles;
        for (uint32_t p = 0; p < 50; ++p) {
            uint32_t r, cc;
            if (!ng.tile_pair(tile, p, r, cc)) continue;
            if (n_pairs < capacity) {
                out[3 * n_pairs] = ng.cand(r);
                out[3 * n_pairs + 1] = ng.cand(cc);
                out[3 * n_pairs + 2] = ((tile >> 22) & 3u) == kKindF;
            }
            ++n_pairs;
        }
    };
    for (uint32_t t = 0; t < ng.f_tiles(); ++t) emit(ng.f_tile(0, t));
    for (uint32_t t = 0; t < ng.u_tiles(); ++t) emit(ng.u_tile(0, t));
    for (uint32_t t = 0; t < ng.t_tiles(); ++t) emit(ng.t_tile(0, t));
    *count = n_pairs;
    return int(n_tiles);
}
