// The local join (compute_step, reference descent.hpp:82-153) on sm_100a, in
// two stages per iteration.
//
// 1. join_distances_kernel — the FP32 hot loop.  One CTA (128 threads = 16
//    groups of 8) evaluates, for one active node u at a time, every
//    new x new unordered pair and every new x old pair of u's candidate lists
//    (the same C(nn,2) + nn*no evaluations as compute_step) and writes the
//    proposals that can matter to u's proposal block in HBM.  Candidate rows stream through shared
//    memory in 32-float slabs (cp.async, double-buffered); each group owns an
//    8x8 pair tile, thread l8 of the group being reference lane l8.
// 2. join_merge_kernel — the bounded list updates.  One warp per target t
//    walks the reverse index (every (u, position) whose lists name t), reads
//    t's row of each proposal block, and inserts the partners that beat t's
//    current maximum into t's sorted row with try_insert's semantics
//    (graph.hpp:116-129: strict improvement, id dedup, evict the max).  A
//    target is owned by exactly one warp, so there are no locks and no
//    atomics on graph rows; the result is the reference's (the k smallest
//    distinct candidates, order-invariant up to exact ties).
//
// Distances are bit-identical to the reference's compiled kernels.  The
// reference sums (a_j - b_j)^2 in eight strided lanes (lane l owns elements
// 8c + l) and reduces them as ((0+1)+(2+3))+((4+5)+(6+7)) (distance.hpp:29-51).
// Pairs inside a full 5x5 or triangular tile (block_core / tri_core5) are
// accumulated with a fused multiply-add, the rest (remainder rows of
// mutual_block_distances, partial new x old tiles) unfused (
// pinned in tests/test_oracle_pins.py).  Rows and columns of u's pair matrix
// are laid out in "slots" so that every 8x8 tile is entirely fused or entirely
// unfused: rows = [new 0..fullN) pad8 [new fullN..nn) pad8, columns =
// [new 0..fullN) [old 0..fullO) pad8 [new fullN..nn) [old fullO..no) pad8,
// with fullN = nn - nn%5, fullO = no - no%5.  Zero padding of the last slab is
// exact (0 - 0 contributes +0 to either form).
//
// Proposal block of u (nn new, no old, m = nn + no candidates),
// nn*(m + no) + no u64 words at doff[u], one row per candidate (prow below):
// row r < nn (new r) has m words, row r >= nn (old r - nn) has nn + 1.  Word 0
// is the row's count, then that many keys (distance bits << 32 | partner id):
// every evaluated pair is a proposal to both endpoints, kept only when it
// beats the endpoint's iteration-start row maximum (c.filter; rows maxima only
// fall during an iteration, so the filter never drops an accepted update).
#include <cstdio>
#include <cstdlib>
#include <cub/device/device_scan.cuh>

#include "kernels.cuh"
#include "tile_math.cuh"

namespace knng_cuda {

namespace {

#ifndef KNNG_JOIN_THREADS
#define KNNG_JOIN_THREADS 128
#endif
constexpr uint32_t kThreads = KNNG_JOIN_THREADS;  // 128: 4 warps, 16 groups of 8 lanes
constexpr uint32_t kGroups = kThreads / 8;
#ifndef KNNG_JOIN_SLAB
#define KNNG_JOIN_SLAB 32
#endif
#ifndef KNNG_JOIN_STAGES
#define KNNG_JOIN_STAGES 3
#endif
constexpr uint32_t kSlab = KNNG_JOIN_SLAB;      // floats per row per smem stage
constexpr uint32_t kStages = KNNG_JOIN_STAGES;  // cp.async pipeline depth
constexpr uint32_t kMaxM = 2 * kMaxCap;  // candidates per node
constexpr uint32_t kMaxRowSlots = kMaxCap + 16;
constexpr uint32_t kMaxColSlots = kMaxM + 16;  // column slots of one node
constexpr uint16_t kDeadTile = 0xffffu;
constexpr uint32_t kInvalid = 0xffu;

// Candidate rows are staged in COLUMN-slot order (every candidate has a column
// slot; a new candidate's row slot maps to a column slot of the same 8-block
// offset, see a_blk below), 32 floats per row per stage.  The four 8-float
// segments of a row are XOR-swizzled by the row's 8-block index so that the
// four 8-lane groups of a warp, reading the same element of rows from
// different 8-blocks, hit four different bank octets.
//
// A CTA works on a BATCH of active nodes (up to kMaxBatch) whose column
// slots share one slot table.  Two staging modes, chosen per launch:
//  - pass mode (long rows): each pass of up to 16 tiles (one per 8-lane
//    group) stages only the 8-blocks its tiles read — at most kPassBlk, packed
//    into ring positions — slab by slab through a kStages-deep cp.async ring.
//    The ring is sized by kPassBlk, not by the batch, so a batch can hold
//    many nodes and passes stay full across node boundaries.
//  - resident mode (short rows, all slabs fit): the batch's rows are staged
//    once, slab s of slot r at ring row s * res_slots + r, and every pass
//    reads them without further staging.
constexpr uint32_t kMaxBatch = 8;              // nodes per CTA batch
constexpr uint32_t kSlotTab = 320;             // batch column slots (pass mode budget)
constexpr uint32_t kBlkTab = kSlotTab / 8;     // batch 8-blocks
#ifndef KNNG_JOIN_PASSBLK
#define KNNG_JOIN_PASSBLK 15
#endif
constexpr uint32_t kPassBlk = KNNG_JOIN_PASSBLK;  // 8-blocks one pass may stage
constexpr uint32_t kRingRows = kPassBlk * 8;   // rows per ring stage
// an 8-block of rows in a ring stage: 8 rows of kSlab floats plus 8 floats of
// padding, so the four groups of a warp reading the same element of rows
// from four consecutive blocks hit four different bank octets
constexpr uint32_t kBlkPitch = 8 * kSlab + 8;
constexpr uint32_t kMaxTiles = 512;            // tiles of one batch
static_assert(kMaxColSlots <= kSlotTab, "one node must fit the slot table");
static_assert(kBlkTab <= 64, "pass block masks are 64-bit");
static_assert(kPassBlk >= 8, "a warp's four tiles may read eight 8-blocks");

struct DistShared {
    // the slab ring (kStages x kPassBlk x kBlkPitch floats) follows this
    // struct in dynamic shared memory
    uint32_t colrow[kSlotTab];                // batch col slot -> data row id (~0: padding)
    float colmax[kSlotTab];                   // batch col slot -> candidate's row maximum
    uint32_t rowcnt[kSlotTab];                // proposals kept per candidate row, at colbase + r
    uint8_t colmap[kSlotTab];                 // batch col slot -> combined index in its node
    uint8_t rowmap[kMaxBatch][kMaxRowSlots];  // row slot -> new index, per node
    uint16_t tiles[kMaxTiles];                // (node << 13) | (rb << 8) | cb
    uint8_t blkpos[kBlkTab];                  // pass mode: batch 8-block -> ring position
    uint8_t blklist[kPassBlk];                // pass mode: ring position -> batch 8-block
    uint32_t ringrow[kRingRows];              // pass mode: ring row -> data row (~0: none)
    uint32_t n_tiles, pass_len, nblk, slot_budget;
    // claimed-but-unbatched nodes (claims come in chunks of kMaxBatch)
    uint32_t qn;
    uint4 q[2 * kMaxBatch];  // active-node records (scatter_rev_kernel)
    uint32_t warp_cnt[kThreads / 32];
    // batch descriptors, double-buffered: warp 0 forms the next batch while
    // the current one is processed
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
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;\n" ::); }

constexpr size_t kSlabOffset = (sizeof(DistShared) + 127) / 128 * 128;
constexpr size_t kDistSmem = kSlabOffset + size_t(kStages) * kPassBlk * kBlkPitch * sizeof(float);
#ifndef KNNG_JOIN_MINBLOCKS
#define KNNG_JOIN_MINBLOCKS 4
#endif
// KNNG_JOIN_MINBLOCKS CTAs per SM: shared memory within the SM's 228 KB
// (1 KB reserved per CTA); registers capped by __launch_bounds__
static_assert(kDistSmem + 1024 <= 228 * 1024 / KNNG_JOIN_MINBLOCKS,
              "join distance kernel shared memory over budget");

__device__ __forceinline__ float* ring_base(DistShared& sh) {
    return reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(&sh) + kSlabOffset);
}

// Float offset of row x of 8-block blk within a ring stage.
__device__ __forceinline__ uint32_t ring_row(uint32_t blk, uint32_t x) {
    return blk * kBlkPitch + x * kSlab;
}

// Resident mode: every column slot of the batch, all slabs, staged once;
// slab s of slot r at ring row s * res_slots + r (res_slots a multiple of 8).
// kSlab / 4 consecutive threads take the 16-byte chunks of one row slab, so
// each row slab is one coalesced read; chunks past the row stride are never
// read.
__device__ __forceinline__ void stage_batch(DistShared& sh, const float* __restrict__ data,
                                            uint32_t stride, uint32_t nslots, uint32_t n_slabs,
                                            uint32_t res_slots) {
    constexpr uint32_t kC4 = kSlab / 4;  // 16-byte chunks per row slab
    const uint32_t j = threadIdx.x % kC4;
    float* ring = ring_base(sh);
    for (uint32_t s = 0; s < n_slabs; ++s) {
        const uint32_t e = s * kSlab + 4 * j;
        if (e >= stride) continue;
        float* const slab = ring + size_t(s) * (res_slots / 8) * kBlkPitch + 4 * j;
        for (uint32_t slot = threadIdx.x / kC4; slot < nslots; slot += kThreads / kC4) {
            const uint32_t row = sh.colrow[slot];
            if (row != 0xffffffffu)
                cp_async16(slab + ring_row(slot >> 3, slot & 7u), data + size_t(row) * stride + e);
        }
    }
}

// One 32-float slab of an 8x8 pair tile: rows of A-block a_blk against rows of
// B-block b_blk; lane l8 accumulates elements 8 s + l8 (reference lane l8).
// The packed FP32x2 pipe (FFMA2 / FMUL2 / FADD2, sm_100) evaluates two pairs
// per instruction, each element with the scalar instruction's IEEE rounding:
// diff = fma(b, -1, a) == a - b exactly (b * -1 is exact, one rounding), then
// acc = fma(diff, diff, acc) on fused tiles or acc + (diff * diff) on unfused
// ones.  acc[4 x + j] holds pairs (x, 2j) and (x, 2j + 1).
template <bool kFusedTile>
__device__ __forceinline__ void tile_slab(const float* __restrict__ slab, uint32_t a_blk,
                                          uint32_t b_blk, uint32_t l8, uint32_t nseg,
                                          float2 minus_zero, float2 (&acc)[32]) {
    const float2 minus_one = make_float2(-1.0f, -1.0f);
#pragma unroll
    for (uint32_t s = 0; s < kSlab / 8; ++s) {
        if (s >= nseg) break;  // the row's last slab may be partial (stride % 32)
        const float* pa = slab + ring_row(a_blk, 0) + 8 * s + l8;
        const float* pb = slab + ring_row(b_blk, 0) + 8 * s + l8;
        float a[8];
        float2 b[4];
#pragma unroll
        for (uint32_t x = 0; x < 8; ++x) a[x] = pa[x * kSlab];
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) {
            b[j].x = pb[(2 * j) * kSlab];
            b[j].y = pb[(2 * j + 1) * kSlab];
        }
#pragma unroll
        for (uint32_t x = 0; x < 8; ++x) {
            const float2 ax = make_float2(a[x], a[x]);
#pragma unroll
            for (uint32_t j = 0; j < 4; ++j) {
                const float2 diff = __ffma2_rn(b[j], minus_one, ax);
                if (kFusedTile)
                    acc[4 * x + j] = __ffma2_rn(diff, diff, acc[4 * x + j]);
                else
                {
                    // unfused: the rounded square as fma(diff, diff, -0) (x + -0
                    // == x exactly, +0 included), then a packed FADD2.  ptxas
                    // (CUDA 12.9) contracts a packed mul.rn.f32x2 +
                    // add.rn.f32x2 pair into FFMA2 even under --fmad=false, and
                    // turns an fma with a literal -0 addend into that mul, so
                    // the -0 arrives as a kernel argument it cannot see
                    // through (checked in SASS and by the bit-exact tests).
                    const float2 sq = __ffma2_rn(diff, diff, minus_zero);
                    acc[4 * x + j] = __fadd2_rn(acc[4 * x + j], sq);
                }
            }
        }
    }
}

// One 32-float slab of a U tile: the (at most 4) leftover new rows of a node
// — rows 0..3 of A-block a_blk — against 16 columns, the rows of B-blocks
// b_blk and b2_blk.  Leftover rows pair only through the reference's
// flexible paths, so every pair is unfused.  acc[8 x + j] holds pairs
// (x, 2j) and (x, 2j + 1), j < 4 in b_blk and j >= 4 in b2_blk; after
// group_reduce64 the lane holding row X has pairs (X / 2, 8 (X % 2) + y),
// i.e. one whole column block.  A node with nn = 4, no = 26 takes two U tiles
// instead of four 8 x 8 tiles with half their rows empty.
__device__ __forceinline__ void tile_slab_u(const float* __restrict__ slab, uint32_t a_blk,
                                            uint32_t b_blk, uint32_t b2_blk, uint32_t l8,
                                            uint32_t nseg, float2 minus_zero, float2 (&acc)[32]) {
    const float2 minus_one = make_float2(-1.0f, -1.0f);
#pragma unroll
    for (uint32_t s = 0; s < kSlab / 8; ++s) {
        if (s >= nseg) break;
        const float* pa = slab + ring_row(a_blk, 0) + 8 * s + l8;
        const float* pb = slab + ring_row(b_blk, 0) + 8 * s + l8;
        const float* pc = slab + ring_row(b2_blk, 0) + 8 * s + l8;
        float a[4];
        float2 b[8];
#pragma unroll
        for (uint32_t x = 0; x < 4; ++x) a[x] = pa[x * kSlab];
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) {
            b[j].x = pb[(2 * j) * kSlab];
            b[j].y = pb[(2 * j + 1) * kSlab];
            b[4 + j].x = pc[(2 * j) * kSlab];
            b[4 + j].y = pc[(2 * j + 1) * kSlab];
        }
#pragma unroll
        for (uint32_t x = 0; x < 4; ++x) {
            const float2 ax = make_float2(a[x], a[x]);
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
                const float2 diff = __ffma2_rn(b[j], minus_one, ax);
                const float2 sq = __ffma2_rn(diff, diff, minus_zero);  // see tile_slab
                acc[8 * x + j] = __fadd2_rn(acc[8 * x + j], sq);
            }
        }
    }
}

// Per-node slot geometry (see the file comment): fullN/fullO, the padded
// fused/unfused row and column extents, and the slot -> index maps.
// kContig (the U-tile kernel): with no fused rows (nn < 5) no pair is fused,
// so the columns are laid out contiguously, [new | old], instead of fused ++
// leftover blocks.
template <bool kContig>
struct NodeGeomT {
    uint32_t nn, no, fn, fo, rf, rs, cf, cs;
    __device__ __forceinline__ void set(uint32_t nn_, uint32_t no_) {
        nn = nn_;
        no = no_;
        fn = nn - nn % 5;
        fo = (fn || !kContig) ? no - no % 5 : 0u;
        rf = (fn + 7) & ~7u;
        rs = (nn - fn + 7) & ~7u;
        cf = (fn + fo + 7) & ~7u;
        cs = (nn - fn + no - fo + 7) & ~7u;
    }
    __device__ __forceinline__ uint32_t rbs() const { return (rf + rs) / 8; }
    __device__ __forceinline__ uint32_t cbs() const { return (cf + cs) / 8; }
    // U tiles (4 x 16, see tile_slab_u): the leftover-row block rf / 8 against
    // column-block pairs (2p, 2p + 1); only when there are leftover rows
    __device__ __forceinline__ uint32_t uts() const { return rs ? (cbs() + 1) / 2 : 0u; }
    __device__ __forceinline__ uint32_t row(uint32_t sl) const {  // row slot -> new index
        if (sl < fn) return sl;
        if (sl >= rf && sl - rf < nn - fn) return fn + (sl - rf);
        return kInvalid;
    }
    __device__ __forceinline__ uint32_t col(uint32_t sl) const {  // col slot -> combined index
        if (sl < fn) return sl;
        if (sl < fn + fo) return nn + (sl - fn);
        if (sl >= cf && sl - cf < nn - fn) return fn + (sl - cf);
        if (sl >= cf + (nn - fn) && sl - cf - (nn - fn) < no - fo)
            return nn + fo + (sl - cf - (nn - fn));
        return kInvalid;
    }
};

#ifndef KNNG_JOIN_PREFETCH
#define KNNG_JOIN_PREFETCH 1
#endif
#ifndef KNNG_JOIN_CHECKS
#define KNNG_JOIN_CHECKS 0  // 1: device-side bounds checks with a message (diagnostics)
#endif
#if KNNG_JOIN_CHECKS
#define JCHECK(cond, what, a, b)                                                        \
    do {                                                                                \
        if (!(cond)) {                                                                  \
            printf("join check failed: %s (%u, %u) block %d thread %d\n", what,        \
                   unsigned(a), unsigned(b), int(blockIdx.x), int(threadIdx.x));      \
            __trap();                                                                   \
        }                                                                               \
    } while (0)
#else
#define JCHECK(cond, what, a, b) ((void)0)
#endif
#ifndef KNNG_JOIN_STATS
#define KNNG_JOIN_STATS 0  // 1: count batches / passes / tiles / staged blocks (diagnostics)
#endif
#if KNNG_JOIN_STATS
__device__ unsigned long long g_join_stats[8];
#define JOIN_STAT(i, v) atomicAdd(&g_join_stats[i], (unsigned long long)(v))
#else
#define JOIN_STAT(i, v) ((void)0)
#endif

// A CTA takes a BATCH of active nodes whose column slots fit the slot budget
// together (up to kMaxBatch nodes), so short lists (late iterations, small k)
// share one tile sweep, one set of barriers and one staging pass instead of
// paying them per node.  res_slots > 0 selects resident mode with that slot
// budget; 0 selects pass mode.
// kU: U tiles (tile_slab_u) for nodes without fused rows — the long-row
// instantiation; the other keeps 8x8 tiles only (see launch_join_distances).
template <bool kU>
__global__ void __launch_bounds__(kThreads, KNNG_JOIN_MINBLOCKS) join_distances_kernel(
    GraphView g, CandView c, const uint32_t* __restrict__ active, IterCounters* ctr,
    uint32_t res_slots, float minus_zero) {
    using NodeGeom = NodeGeomT<kU>;
    constexpr bool utiles = kU;
    const float2 mz2 = make_float2(minus_zero, minus_zero);  // -0.0f, opaque to ptxas
    extern __shared__ __align__(128) unsigned char smem_raw[];
    DistShared& sh = *reinterpret_cast<DistShared*>(smem_raw);
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
    uint32_t gslab = 0;  // pass mode: slabs staged so far (ring stage = gslab % kStages)
    // warp 0 claims chunks of kMaxBatch active indices one batch ahead, so
    // the claim's atomic round trip overlaps the current batch
    uint32_t a_next = 0;
    if (tid == 0) a_next = atomicAdd(&ctr->work, kMaxBatch);

    // warp 0 forms a batch into D: top the queue up with the claimed chunk
    // (one 16-byte record per node), claim the next, then take the longest
    // queue prefix whose column slots and tiles fit
    auto form_batch = [&](DistShared::Batch& D) {
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
            NodeGeom ng;
            ng.set(nn, no);
            s_l = ng.cf + ng.cs;
            t_l = ng.rbs() * ng.cbs();
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
            if (nv == 0) D.nslots = 0;  // no stale slots for the prefetch
        }
    };
    // Column-slot contents of batch D, kSlotsPerThread slots per thread
    // (slot s = tid + kThreads j): the candidate's data-row id and row
    // maximum.  Loaded into registers one batch ahead, so the loads are in
    // flight while the current batch computes.
    constexpr uint32_t kSlotsPerThread = (kSlotTab + kThreads - 1) / kThreads;
    uint32_t pf_id[kSlotsPerThread];
    float pf_max[kSlotsPerThread];
    auto load_slots = [&](const DistShared::Batch& D) {
#pragma unroll
        for (uint32_t j = 0; j < kSlotsPerThread; ++j) {
            const uint32_t sidx = tid + kThreads * j;
            pf_id[j] = 0xffffffffu;
            pf_max[j] = 0.0f;
            if (D.nv > 0 && sidx < D.nslots) {
                uint32_t v = 0;
                while (v + 1 < D.nv && D.colbase[v + 1] <= sidx) ++v;
                NodeGeom ng;
                ng.set(D.vnn[v], D.vno[v]);
                const uint32_t x = ng.col(sidx - D.colbase[v]);
                if (x != kInvalid) {
                    const uint32_t pos = x < ng.nn ? x : cap + x - ng.nn;
                    const size_t base = size_t(D.node[v]) * 2 * cap;
                    pf_id[j] = c.ids[base + pos];
                    pf_max[j] = c.filter ? c.cmax[base + pos] : __int_as_float(0x7f800000);
                }
            }
        }
    };

    uint32_t cur = 0;
    __syncthreads();  // the queue state tid 0 initialised
    if (tid < 32) form_batch(sh.bd[0]);
    __syncthreads();
#if KNNG_JOIN_PREFETCH
    load_slots(sh.bd[0]);
#endif
    while (true) {
        const DistShared::Batch& B = sh.bd[cur];
        const uint32_t nv = B.nv;
        if (nv == 0) break;
        if (tid == 0) {
            JOIN_STAT(0, 1);
            JOIN_STAT(1, nv);
            sh.n_tiles = 0;
        }
        // slot maps of the batch (contents prefetched one batch ahead)
#if !KNNG_JOIN_PREFETCH
        load_slots(B);
#endif
#pragma unroll
        for (uint32_t j = 0; j < kSlotsPerThread; ++j) {
            const uint32_t sidx = tid + kThreads * j;
            if (sidx < B.nslots) {
                uint32_t v = 0;
                while (v + 1 < nv && B.colbase[v + 1] <= sidx) ++v;
                NodeGeom ng;
                ng.set(B.vnn[v], B.vno[v]);
                JCHECK(sidx < kSlotTab && v < nv, "slot map", sidx, v);
                sh.colmap[sidx] = uint8_t(ng.col(sidx - B.colbase[v]));
                sh.colrow[sidx] = pf_id[j];
                sh.colmax[sidx] = pf_max[j];
            }
        }
        for (uint32_t v = 0; v < nv; ++v) {
            NodeGeom ng;
            ng.set(B.vnn[v], B.vno[v]);
            for (uint32_t sl = tid; sl < ng.rf + ng.rs; sl += kThreads)
                sh.rowmap[v][sl] = uint8_t(ng.row(sl));
            for (uint32_t r = tid; r < ng.nn + ng.no; r += kThreads) sh.rowcnt[B.colbase[v] + r] = 0;
        }
        // warp 0 forms the next batch meanwhile
        if (tid < 32) form_batch(sh.bd[cur ^ 1u]);
        __syncthreads();
#if KNNG_JOIN_PREFETCH
        load_slots(sh.bd[cur ^ 1u]);  // consumed by the next iteration
#endif
        // resident mode: the batch's rows load while the tile list is built
        if (resident) {
            stage_batch(sh, g.data, stride, B.nslots, n_slabs, res_slots);
            cp_async_commit();
        }
        // live tiles (any valid pair) of all nodes: fused tiles, padding to a
        // whole warp (4 groups), then unfused tiles, so every warp runs one
        // path; in (node, rb, cb) order so a warp's groups mostly share A
        // (built by warp 0 alone: ballot compaction in chunks of 32, no CTA
        // barriers while the other warps' row copies are in flight)
        if (tid < 32) {
            const uint32_t lane = tid;
            // phase 0: fused 8x8 tiles; 1: unfused 8x8 tiles (with U tiles on:
            // all but the leftover-row block); 2: U tiles.  Each run is padded
            // to whole warps so every warp runs one path.
            // U tiles only for nodes without fused rows (nn < 5: late
            // iterations); they lose to 8x8 tiles when they share a pass with
            // a node's fused tiles (C5 iterations 1-4, measured)
            auto count = [&](const NodeGeom& ng, uint32_t phase) -> uint32_t {
                if (phase == 2) return utiles && ng.fn == 0 ? ng.uts() : 0u;
                return ng.rbs() * ng.cbs();
            };
            uint32_t total01 = 0, total2 = 0;
            for (uint32_t v = 0; v < nv; ++v) {
                NodeGeom ng;
                ng.set(B.vnn[v], B.vno[v]);
                total01 += count(ng, 0);
                total2 += count(ng, 2);
            }
            uint32_t nt = 0;
            for (uint32_t phase = 0; phase < (total2 ? 3u : 2u); ++phase) {
                const uint32_t total = phase == 2 ? total2 : total01;
                for (uint32_t t0 = 0; t0 < total; t0 += 32) {
                    uint32_t t = t0 + lane, v = 0, rb = 0, cb = 0;
                    bool live = false;
                    if (t < total) {
                        NodeGeom ng;
                        ng.set(B.vnn[0], B.vno[0]);
                        while (t >= count(ng, phase)) {
                            t -= count(ng, phase);
                            ++v;
                            ng.set(B.vnn[v], B.vno[v]);
                        }
                        if (phase == 2) {
                            // U tile t: leftover rows x column blocks 2t, 2t + 1
                            rb = ng.rf / 8;
                            cb = 0x80u | t;
                            for (uint32_t y = 0; y < 16 && 16 * t + y < ng.cf + ng.cs; ++y) {
                                const uint32_t col = sh.colmap[B.colbase[v] + 16 * t + y];
                                live |= col != kInvalid && (col >= ng.nn || col > ng.fn);
                            }
                        } else {
                            rb = t / ng.cbs();
                            cb = t % ng.cbs();
                            const bool fused_tile = rb * 8 < ng.rf && cb * 8 < ng.cf;
                            const bool u_row = utiles && ng.fn == 0;  // all its tiles are U tiles
                            if (fused_tile == (phase == 0) && !u_row) {
                                uint32_t imin = kInvalid;
                                for (uint32_t x = 0; x < 8; ++x)
                                    imin = min(imin, uint32_t(sh.rowmap[v][rb * 8 + x]));
                                if (imin != kInvalid)
                                    for (uint32_t y = 0; y < 8; ++y) {
                                        const uint32_t col = sh.colmap[B.colbase[v] + cb * 8 + y];
                                        live |= col != kInvalid && (col >= ng.nn || col > imin);
                                    }
                            }
                        }
                    }
                    const uint32_t mask = __ballot_sync(0xffffffffu, live);
                    if (live)
                        sh.tiles[nt + __popc(mask & ((1u << lane) - 1u))] =
                            uint16_t((v << 13) | (rb << 8) | cb);
                    nt += __popc(mask);
                }
                if (phase == 0 || (phase == 1 && total2)) {  // pad the run to whole warps
                    const uint32_t padded = (nt + 3u) & ~3u;
                    if (lane < padded - nt) sh.tiles[nt + lane] = kDeadTile;
                    nt = padded;
                }
            }
            if (lane == 0) sh.n_tiles = nt;
        }
        if (resident) cp_async_wait_0();
        __syncthreads();
        const uint32_t n_tiles = sh.n_tiles;
        if (tid == 0) JOIN_STAT(6, n_tiles);

        uint32_t pass_len = kGroups;
        for (uint32_t t0 = 0; t0 < n_tiles; t0 += pass_len) {
            if (resident && tid == 0) {
                JOIN_STAT(2, 1);
                JOIN_STAT(3, min(kGroups, n_tiles - t0));
            }
            if (!resident) {
                // warp 0 schedules the pass: the longest run of whole warps'
                // tiles (<= 16) whose 8-blocks fit kPassBlk ring positions
                if (tid < 32) {
                    const uint32_t lane = tid, left = min(kGroups, n_tiles - t0);
                    uint64_t m = 0;
                    if (lane < left) {
                        const uint32_t tile = sh.tiles[t0 + lane];
                        if (tile != kDeadTile) {
                            const uint32_t v = tile >> 13, rb = (tile >> 8) & 31u,
                                           cb = tile & 0xffu;
                            NodeGeom ng;
                            ng.set(B.vnn[v], B.vno[v]);
                            const uint32_t cb0 = B.colbase[v] / 8;
                            const uint32_t ab =
                                cb0 + (rb * 8 < ng.rf ? rb : ng.cf / 8 + (rb - ng.rf / 8));
                            if (kU && (cb & 0x80u)) {  // U tile: column blocks 2t, 2t + 1
                                const uint32_t c0 = 2 * (cb & 0x7fu);
                                m = (1ull << ab) | (1ull << (cb0 + c0));
                                if (c0 + 1 < ng.cbs()) m |= 1ull << (cb0 + c0 + 1);
                            } else {
                                m = (1ull << ab) | (1ull << (cb0 + cb));
                            }
                        }
                    }
#pragma unroll
                    for (uint32_t o = 1; o < 32; o <<= 1) {
                        const uint64_t mp = __shfl_up_sync(0xffffffffu, m, o);
                        if (lane >= o) m |= mp;
                    }
                    const bool ok = lane < left && __popcll(m) <= kPassBlk &&
                                    ((lane & 3u) == 3u || lane + 1 == left);
                    const uint32_t okm = __ballot_sync(0xffffffffu, ok);
                    const uint32_t last = 31u - __clz(okm);  // 4 tiles need <= 8 blocks
                    const uint64_t pm = __shfl_sync(0xffffffffu, m, last);
                    for (uint32_t bit = lane; bit < kBlkTab; bit += 32)
                        if ((pm >> bit) & 1ull) {
                            const uint32_t pos = __popcll(pm & ((1ull << bit) - 1ull));
                            sh.blkpos[bit] = uint8_t(pos);
                            sh.blklist[pos] = uint8_t(bit);
                        }
                    __syncwarp();
                    // ring row -> data row of the pass (~0: padding slot)
                    const uint32_t nrows = __popcll(pm) * 8u;
                    for (uint32_t r = lane; r < kRingRows; r += 32)
                        sh.ringrow[r] =
                            r < nrows ? sh.colrow[sh.blklist[r >> 3] * 8u + (r & 7u)] : 0xffffffffu;
                    if (lane == 0) {
                        sh.pass_len = last + 1;
                        sh.nblk = __popcll(pm);
                    }
                }
                __syncthreads();
                pass_len = sh.pass_len;
                if (tid == 0) {
                    JOIN_STAT(2, 1);
                    JOIN_STAT(3, pass_len);
                    JOIN_STAT(4, sh.nblk);
                    JOIN_STAT(5, n_slabs);
                }
            }
            const uint32_t t = t0 + group;
            const uint32_t tile0 = group < pass_len && t < n_tiles ? sh.tiles[t] : kDeadTile;
            const bool live = tile0 != kDeadTile;
            const uint32_t tile = live ? tile0 : 0u;
            const uint32_t v = tile >> 13, rb = (tile >> 8) & 31u;
            const bool utile = kU && (tile & 0x80u) != 0u;
            NodeGeom ng;
            ng.set(B.vnn[v], B.vno[v]);
            // 8x8 tiles: column block cb; U tiles: blocks 2t and 2t + 1
            const uint32_t cb = utile ? 2u * (tile & 0x7fu) : (tile & 0xffu);
            const bool cb2_ok = utile && cb + 1 < ng.cbs();
            const bool fused = !utile && rb * 8 < ng.rf && cb * 8 < ng.cf;
            // row slot block -> column slot block holding the same new
            // candidates, then into the batch's column-slot space
            const uint32_t cb0 = B.colbase[v] / 8;
            const uint32_t a_blk = cb0 + (rb * 8 < ng.rf ? rb : ng.cf / 8 + (rb - ng.rf / 8));
            const uint32_t b_blk = cb0 + cb;
            const uint32_t b2_blk = cb2_ok ? b_blk + 1 : b_blk;  // past the node: ignored
            float2 acc[32];
#pragma unroll
            for (uint32_t p = 0; p < 32; ++p) acc[p] = make_float2(0.0f, 0.0f);
            if (resident) {
                if (live)
                    for (uint32_t s = 0; s < n_slabs; ++s) {
                        const float* slab = ring_base(sh) + size_t(s) * (res_slots / 8) * kBlkPitch;
                        const uint32_t nseg = min(kSlab, stride - s * kSlab) / 8u;
                        if (utile)
                            tile_slab_u(slab, a_blk, b_blk, b2_blk, l8, nseg, mz2, acc);
                        else if (fused)
                            tile_slab<true>(slab, a_blk, b_blk, l8, nseg, mz2, acc);
                        else
                            tile_slab<false>(slab, a_blk, b_blk, l8, nseg, mz2, acc);
                    }
            } else {
                const uint32_t a_pos = live ? sh.blkpos[a_blk] : 0u;
                const uint32_t b_pos = live ? sh.blkpos[b_blk] : 0u;
                const uint32_t b2_pos = live && cb2_ok ? sh.blkpos[b2_blk] : b_pos;
                // kStages-deep cp.async ring, one barrier per slab.  Thread
                // tid stages 16-byte chunk tid % kC4 of ring rows
                // tid / kC4 + kSweep q; its data rows are read from the ring
                // table once per pass.
                constexpr uint32_t kC4 = kSlab / 4, kSweep = kThreads / kC4;
                constexpr uint32_t kRowsPerThread = (kRingRows + kSweep - 1) / kSweep;
                static_assert(kSweep % 8 == 0, "a sweep covers whole 8-blocks");
                const uint32_t j = tid % kC4, r0 = tid / kC4;
                uint32_t my_rows[kRowsPerThread];
#pragma unroll
                for (uint32_t q = 0; q < kRowsPerThread; ++q) {
                    const uint32_t r = r0 + kSweep * q;
                    my_rows[q] = r < kRingRows ? sh.ringrow[r] : 0xffffffffu;
                }
                float* const my_dst = ring_base(sh) + ring_row(r0 >> 3, r0 & 7u) + 4 * j;
                auto issue = [&](uint32_t sl) {
                    const uint32_t st = (gslab + sl) % kStages, e = sl * kSlab + 4 * j;
                    if (e < stride) {
                        float* const dst = my_dst + size_t(st) * kPassBlk * kBlkPitch;
#pragma unroll
                        for (uint32_t q = 0; q < kRowsPerThread; ++q)
                            if (my_rows[q] != 0xffffffffu)
                                cp_async16(dst + q * (kSweep / 8) * kBlkPitch,
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
                    const float* slab = ring_base(sh) + size_t(st) * kPassBlk * kBlkPitch;
                    const uint32_t nseg = min(kSlab, stride - sl * kSlab) / 8u;
                    if (live) {
                        if (utile)
                            tile_slab_u(slab, a_pos, b_pos, b2_pos, l8, nseg, mz2, acc);
                        else if (fused)
                            tile_slab<true>(slab, a_pos, b_pos, l8, nseg, mz2, acc);
                        else
                            tile_slab<false>(slab, a_pos, b_pos, l8, nseg, mz2, acc);
                    }
                }
                gslab += n_slabs;
            }
            float row[8];
            group_reduce64(acc, l8, row);
            const uint32_t X = reduced_row(l8);
            // this lane's 8 pairs: row slot rb * 8 + x against column block cbx
            const uint32_t x = utile ? X >> 1 : X;
            const uint32_t cbx = utile ? cb + (X & 1u) : cb;
            const bool col_ok = !utile || (X & 1u) == 0u || cb2_ok;
            const uint32_t i = live && col_ok ? sh.rowmap[v][rb * 8 + x] : kInvalid;
            if (i != kInvalid) {
                // each pair is a proposal to both endpoints; kept (compacted
                // into the endpoint's row) only if it beats that candidate's
                // iteration-start row maximum — the stale-upwards prefilter of
                // compute_step (descent.hpp:97-102,134-147)
                const uint32_t nn = ng.nn, m = ng.nn + ng.no;
                uint64_t* const D = c.D + B.doff[v];
                const uint32_t slot_i = B.colbase[v] + (i < ng.fn ? i : ng.cf + (i - ng.fn));
                const uint32_t id_i = sh.colrow[slot_i];
                const float mx_i = sh.colmax[slot_i];
#pragma unroll
                for (uint32_t y = 0; y < 8; ++y) {
                    const uint32_t slot_c = B.colbase[v] + cbx * 8 + y;
                    const uint32_t col = sh.colmap[slot_c];
                    if (col == kInvalid || !(col >= nn || col > i)) continue;
                    // an id listed twice pairs with itself: try_insert ignores
                    // self (graph.hpp:116-129), so neither endpoint gets it
                    // (the unfiltered distances-only entry keeps every pair)
                    if (c.filter && sh.colrow[slot_c] == id_i) continue;
                    const float dist = row[y];
                    if (dist < mx_i) {
                        JCHECK(B.colbase[v] + i < kSlotTab, "rowcnt i", B.colbase[v], i);
                    const uint32_t pos = atomicAdd(&sh.rowcnt[B.colbase[v] + i], 1u);
                    JCHECK(pos + 1 < (i < nn ? m : nn + 1), "row overflow i", pos, m);
                        D[prow(i, nn, m) + 1 + pos] = pack_key(dist, sh.colrow[slot_c]);
                    }
                    if (dist < sh.colmax[slot_c]) {
                        JCHECK(B.colbase[v] + col < kSlotTab, "rowcnt col", B.colbase[v], col);
                    const uint32_t pos = atomicAdd(&sh.rowcnt[B.colbase[v] + col], 1u);
                    JCHECK(pos + 1 < (col < nn ? m : nn + 1), "row overflow col", pos, m);
                        D[prow(col, nn, m) + 1 + pos] = pack_key(dist, id_i);
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


// Warp-wide bounded insert into a sorted row held one key per lane (lanes
// >= k hold kEmptyKey).  try_insert semantics (graph.hpp:116-129).
// Deterministic mode (det): a present id takes the smaller of its two
// distances (the same pair evaluated in two joins; the reference keeps
// whichever its sequential order offered first), and `fresh` marks only ids
// absent from the target's initial row (lane i's initial id: init_id), so the
// final row and its change count do not depend on the insertion order.
__device__ __forceinline__ bool warp_try_insert(uint64_t& key, uint32_t& flags, uint32_t k,
                                                float dist, uint32_t cand,
                                                uint32_t* fresh = nullptr, bool det = false,
                                                uint32_t init_id = 0xffffffffu) {
    const uint32_t lane = lane_id();
    const uint64_t max_key = __shfl_sync(0xffffffffu, key, k - 1);
    if (!(dist < key_dist(max_key))) return false;
    const uint32_t kmask = k >= 32 ? 0xffffffffu : ((1u << k) - 1u);
    const uint64_t nk = pack_key(dist, cand);
    const uint32_t present = __ballot_sync(0xffffffffu, lane < k && key_id(key) == cand);
    if (present) {
        if (!det) return false;
        const uint32_t p = __ffs(present) - 1u;
        if (!(nk < __shfl_sync(0xffffffffu, key, p))) return false;
        // move the entry from p down to its new position pos <= p
        const uint32_t pos = __popc(__ballot_sync(0xffffffffu, lane < k && key < nk));
        const uint64_t up = __shfl_up_sync(0xffffffffu, key, 1);
        if (lane < k) key = (lane < pos || lane > p) ? key : (lane == pos ? nk : up);
        auto carry = [&](uint32_t b) {
            const uint32_t bp = (b >> p) & 1u;
            const uint32_t mid = ((1u << p) - 1u) & ~((1u << pos) - 1u);  // bits [pos, p)
            return ((b & ~(mid | (1u << p))) | ((b & mid) << 1) | (bp << pos)) & kmask;
        };
        flags = carry(flags);
        if (fresh) *fresh = carry(*fresh);
        return true;
    }
    const uint32_t pos = __popc(__ballot_sync(0xffffffffu, lane < k && key < nk));
    const uint64_t up = __shfl_up_sync(0xffffffffu, key, 1);
    if (lane < k) key = lane < pos ? key : (lane == pos ? nk : up);
    const uint32_t low = (1u << pos) - 1u;
    flags = ((flags & low) | (1u << pos) | ((flags & ~low) << 1)) & kmask;
    if (fresh) {
        const uint32_t came = det ? (__ballot_sync(0xffffffffu, init_id == cand) == 0u) : 1u;
        *fresh = ((*fresh & low) | (came << pos) | ((*fresh & ~low) << 1)) & kmask;
    }
    return true;
}

constexpr uint32_t kMergeWarps = 8;
#ifndef KNNG_MERGE_META
#define KNNG_MERGE_META 2
#endif
constexpr uint32_t kMergeMeta = KNNG_MERGE_META;  // reverse-index chunks per metadata round trip
#ifndef KNNG_MERGE_DEPTH
#define KNNG_MERGE_DEPTH 1
#endif
constexpr uint32_t kMergeDepth = KNNG_MERGE_DEPTH;  // proposal steps fetched ahead

// Merges the proposals of t's reverse-index entries rv[0, cnt) into the row
// held by the calling warp (lane i = entry i).  `fresh` tracks which entries
// came in (shifted like the flags).
template <bool kDet>
__device__ __forceinline__ void merge_entries(const CandView& c, const uint64_t* rv, uint32_t cnt,
                                              uint32_t k, uint64_t& key, uint32_t& flags,
                                              uint32_t& fresh, float& cur_max,
                                              uint32_t& inserted, uint32_t init_id) {
    const uint32_t lane = lane_id();
    // Metadata of kMergeMeta chunks of 32 entries at once, one entry per lane
    // per chunk: where t's row of the node's proposal block starts and how
    // many proposals it kept.  Loading several chunks per round trip matters
    // for hub targets named by thousands of lists, most of whose rows the
    // prefilter left empty.
    for (uint32_t g0 = 0; g0 < cnt; g0 += 32 * kMergeMeta) {
        uint64_t mrows[kMergeMeta];
        uint32_t pes[kMergeMeta];
#pragma unroll
        for (uint32_t q = 0; q < kMergeMeta; ++q) {
            const uint32_t e = g0 + 32 * q + lane;
            mrows[q] = e < cnt ? rv[e] : 0ull;
        }
#pragma unroll
        for (uint32_t q = 0; q < kMergeMeta; ++q) {
            const uint32_t e = g0 + 32 * q + lane;
            pes[q] = e < cnt ? uint32_t(c.D[mrows[q]]) : 0u;
            JCHECK(pes[q] <= 2 * c.cap, "merge row count", e, pes[q]);
        }
#pragma unroll
        for (uint32_t q = 0; q < kMergeMeta; ++q) {
            if (g0 + 32 * q >= cnt) break;
            const uint64_t mrow = mrows[q];
            const uint32_t pe = pes[q];
            // The chunk's proposals, flattened across entries so every lane of
            // every step has work even when rows are short.  Each step's loads
            // are issued one step ahead so the fetch overlaps the inserts.
            uint32_t incl = pe;
#pragma unroll
            for (uint32_t o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const uint32_t excl = incl - pe;
            const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
            struct Step {
                float dist;
                uint32_t cand;
                bool valid;
            };
            auto fetch = [&](uint32_t f0) {
                const uint32_t f = f0 + lane;
                // entry holding flattened partner f: last e with excl[e] <= f
                uint32_t e = 0;
#pragma unroll
                for (uint32_t step = 16; step > 0; step >>= 1) {
                    const uint32_t probe = __shfl_sync(0xffffffffu, excl, (e + step) & 31u);
                    if (e + step < 32 && probe <= f) e += step;
                }
                const uint64_t row = __shfl_sync(0xffffffffu, mrow, e);
                const uint32_t qq = f - __shfl_sync(0xffffffffu, excl, e);
                Step st{0.0f, 0u, f < total};
                if (st.valid) {
                    const uint64_t kk = c.D[row + 1 + qq];
                    st.dist = key_dist(kk);
                    st.cand = key_id(kk);
                }
                return st;
            };
            // kMergeDepth steps of proposals in flight
            Step ring[kMergeDepth];
#pragma unroll
            for (uint32_t q = 0; q < kMergeDepth; ++q)
                ring[q] = 32 * q < total ? fetch(32 * q) : Step{0.0f, 0u, false};
            for (uint32_t f0 = 0; f0 < total; f0 += 32) {
                const Step cur = ring[0];
#pragma unroll
                for (uint32_t q = 0; q + 1 < kMergeDepth; ++q) ring[q] = ring[q + 1];
                ring[kMergeDepth - 1] = f0 + 32 * kMergeDepth < total ? fetch(f0 + 32 * kMergeDepth)
                                                                     : Step{0.0f, 0u, false};
                uint32_t pass = __ballot_sync(0xffffffffu, cur.valid && cur.dist < cur_max);
                while (pass) {
                    const uint32_t src = __ffs(pass) - 1u;
                    pass &= pass - 1u;
                    const float dd = __shfl_sync(0xffffffffu, cur.dist, src);
                    const uint32_t cc = __shfl_sync(0xffffffffu, cur.cand, src);
                    if (dd < cur_max &&
                        warp_try_insert(key, flags, k, dd, cc, &fresh, kDet, init_id)) {
                        ++inserted;
                        cur_max = key_dist(__shfl_sync(0xffffffffu, key, k - 1));
                    }
                }
            }
        }
    }
}

// Incremental in-degree (CandView::indeg_inc): the ids that left row t
// (initial row key0) lose one, the ids that came in (final row key) gain one.
__device__ __forceinline__ void indeg_update(uint32_t* indeg, uint64_t key0, uint64_t key,
                                             uint32_t k) {
    const uint32_t lane = lane_id();
    const uint32_t id0 = lane < k ? key_id(key0) : 0xffffffffu;
    const uint32_t id1 = lane < k ? key_id(key) : 0xfffffffeu;
    bool kept = false, had = false;
    for (uint32_t j = 0; j < k; ++j) {
        kept |= __shfl_sync(0xffffffffu, id1, j) == id0;
        had |= __shfl_sync(0xffffffffu, id0, j) == id1;
    }
    if (lane < k && !kept) atomicSub(indeg + id0, 1u);
    if (lane < k && !had) atomicAdd(indeg + id1, 1u);
}

// Targets named by more than kHubEntries reverse-index entries are left to
// hub_merge_kernel (a whole CTA per target).
#ifndef KNNG_MERGE_MINBLOCKS
#define KNNG_MERGE_MINBLOCKS 8
#endif
#ifndef KNNG_HUB_ENTRIES
#define KNNG_HUB_ENTRIES 256
#endif
constexpr uint32_t kHubEntries = KNNG_HUB_ENTRIES;

template <bool kDet>
__global__ void __launch_bounds__(kMergeWarps * 32, KNNG_MERGE_MINBLOCKS) join_merge_kernel(GraphView g, CandView c,
                                                                     IterCounters* ctr,
                                                                     uint32_t* hubs) {
    // changes are summed per block without a block barrier (targets are
    // uneven; finished warps leave at once): the last warp out flushes
    __shared__ unsigned long long s_changes;
    __shared__ uint32_t s_done;
    if (ctr->overflow || ctr->halt) return;
    if (threadIdx.x == 0) {
        s_changes = 0;
        s_done = 0;
    }
    __syncthreads();
    const uint32_t lane = lane_id();
    const uint32_t t = g.lo + blockIdx.x * kMergeWarps + (threadIdx.x >> 5);
    const uint32_t k = g.k;
    // the row, its flags and the reverse-index range load together (one
    // round trip), speculatively for targets nothing names
    const bool in_range = t < g.hi;
    const uint32_t cnt = in_range ? c.revcnt[t] : 0u;
    const uint32_t roff = in_range ? c.roff[t] : 0u;
    uint64_t key = in_range && lane < k ? g.keys[size_t(t) * k + lane] : kEmptyKey;
    uint32_t flags = in_range ? g.flags[t] : 0u;
    if (cnt > kHubEntries && hubs) {
        if (lane == 0) hubs[atomicAdd(&ctr->hubs, 1u)] = t;
    } else if (cnt) {
        uint32_t fresh = 0;
        float cur_max = key_dist(__shfl_sync(0xffffffffu, key, k - 1));
        uint32_t inserted = 0;
        const uint32_t init_id = kDet ? key_id(key) : 0xffffffffu;
        const uint64_t key0 = key;
        merge_entries<kDet>(c, c.rev + roff, cnt, k, key, flags, fresh, cur_max, inserted, init_id);
        if (inserted) {
            if (c.indeg_inc && !ctr[1].recount) indeg_update(c.indeg_inc, key0, key, k);
            if (lane < k) g.keys[size_t(t) * k + lane] = key;
            if (lane == 0) {
                g.flags[t] = flags;
                g.maxd[t] = cur_max;
                // deterministic mode: |final row \ initial row| (order-free)
                const uint32_t ch = kDet ? __popc(fresh & (k >= 32 ? 0xffffffffu : ((1u << k) - 1u)))
                                         : inserted;
                if (ch) atomicAdd(&s_changes, (unsigned long long)ch);
            }
        }
    }
    if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(&s_done, 1u) == kMergeWarps - 1) {
            __threadfence_block();
            const unsigned long long ch = atomicAdd(&s_changes, 0ull);
            if (ch) atomicAdd(&ctr->changes, ch);
        }
    }
}

// A hub target per CTA: warp w merges a contiguous slice of the target's
// entries into its own copy of the row; warp 0 then inserts the other warps'
// incoming entries.  The result is the k smallest distinct candidates of the
// row and all proposals, as in one warp (ties aside).  The change count is,
// like join_merge_kernel's, the number of successful inserts of the target's
// proposals (each proposal counted at most once: the warps' slice inserts,
// not warp 0's fold-in); deterministic mode counts the entries that came in
// (the order-free count).
#ifndef KNNG_HUB_WARPS
#define KNNG_HUB_WARPS 16  // 16 measured: C2 merge 2.51 -> 2.23 ms with 256 entries
#endif
constexpr uint32_t kHubWarps = KNNG_HUB_WARPS;  // warps per hub CTA

template <bool kDet>
__global__ void __launch_bounds__(kHubWarps * 32) hub_merge_kernel(GraphView g, CandView c,
                                                                    IterCounters* ctr,
                                                                    const uint32_t* hubs) {
    __shared__ unsigned long long s_keys[kHubWarps][32];
    __shared__ uint32_t s_fresh[kHubWarps];
    __shared__ uint32_t s_ins[kHubWarps];
    if (ctr->overflow || ctr->halt) return;
    const uint32_t lane = lane_id(), w = threadIdx.x >> 5, k = g.k;
    const uint32_t nh = ctr->hubs;
    for (uint32_t h = blockIdx.x; h < nh; h += gridDim.x) {
        const uint32_t t = hubs[h];
        const uint32_t cnt = c.revcnt[t];
        const uint32_t b = uint32_t(uint64_t(cnt) * w / kHubWarps);
        const uint32_t e = uint32_t(uint64_t(cnt) * (w + 1) / kHubWarps);
        uint64_t key = lane < k ? g.keys[size_t(t) * k + lane] : kEmptyKey;
        const uint64_t key0 = key;  // the initial row (incremental in-degree)
        uint32_t flags = g.flags[t], fresh = 0, inserted = 0;
        float cur_max = key_dist(__shfl_sync(0xffffffffu, key, k - 1));
        const uint32_t init_id = kDet ? key_id(key) : 0xffffffffu;
        merge_entries<kDet>(c, c.rev + c.roff[t] + b, e - b, k, key, flags, fresh, cur_max, inserted,
                            init_id);
        s_keys[w][lane] = key;
        if (lane == 0) {
            s_fresh[w] = fresh;
            s_ins[w] = inserted;
        }
        __syncthreads();
        if (w == 0) {
            for (uint32_t o = 1; o < kHubWarps; ++o) {
                const uint32_t fr = s_fresh[o];
                for (uint32_t i = 0; i < k; ++i) {
                    // deterministic mode: every entry (smaller copies of
                    // initial ids carry no fresh bit)
                    if (!((fr >> i) & 1u) && !kDet) continue;
                    const uint64_t pk = s_keys[o][i];
                    const float dd = key_dist(pk);
                    if (dd < cur_max &&
                        warp_try_insert(key, flags, k, dd, key_id(pk), &fresh, kDet, init_id))
                        cur_max = key_dist(__shfl_sync(0xffffffffu, key, k - 1));
                }
            }
            const uint32_t kmask = k >= 32 ? 0xffffffffu : ((1u << k) - 1u);
            const uint32_t came = __popc(fresh & kmask);
            uint32_t ins = 0;
            for (uint32_t o = 0; o < kHubWarps; ++o) ins += s_ins[o];
            const uint32_t ch = kDet ? came : ins;
            if (came || kDet) {
                if (c.indeg_inc && !ctr[1].recount) indeg_update(c.indeg_inc, key0, key, k);
                if (lane < k) g.keys[size_t(t) * k + lane] = key;
                if (lane == 0) {
                    g.flags[t] = flags;
                    g.maxd[t] = cur_max;
                }
            }
            if (lane == 0 && ch) atomicAdd(&ctr->changes, (unsigned long long)ch);
        }
        __syncthreads();
    }
}

// One warp per active node: (u, position) into each named candidate's bucket.
__global__ void scatter_rev_kernel(CandView c, const uint32_t* __restrict__ active,
                                   IterCounters* ctr) {
    const uint32_t a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (a >= ctr->active || ctr->overflow) return;
    const uint32_t u = active[a], lane = lane_id();
    const uint32_t nn = c.nc[u], no = c.oc[u], m = nn + no;
    const uint64_t off = c.doff[u];
    if (lane == 0)  // the distance kernel's per-node record
        c.arec[a] = make_uint4(u, nn | (no << 16), uint32_t(off), uint32_t(off >> 32));
    const uint32_t* list = c.ids + size_t(u) * 2 * c.cap;
    // all of this lane's candidates' cursor atomics in flight at once (m <=
    // 128: up to four per lane), then the reverse-index stores
    constexpr uint32_t kPer = (2 * kMaxCap + 31) / 32;
    uint32_t x[kPer], slot[kPer];
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) {
        const uint32_t p = lane + 32 * q;
        if (p < m) {
            x[q] = p < nn ? list[p] : list[c.cap + p - nn];
            slot[q] = atomicAdd(c.rcur + x[q], 1u);
        }
    }
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) {
        const uint32_t p = lane + 32 * q;
        if (p < m) c.rev[c.roff[x[q]] + slot[q]] = off + prow(p, nn, m);  // t's row of u's block
    }
}

__global__ void check_capacity_kernel(IterCounters* ctr, unsigned long long capacity) {
    ctr->overflow = ctr->dwords > capacity ? 1u : 0u;
}

}  // namespace

size_t join_scan_scratch(uint32_t n) {
    size_t a = 0, b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, (const uint64_t*)nullptr, (uint64_t*)nullptr, int(n));
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr, int(n));
    return a > b ? a : b;
}

void launch_join_offsets(const CandView& c, uint32_t n, uint32_t lo, uint32_t hi, void* scratch,
                         size_t scratch_bytes, cudaStream_t s) {
    // proposal blocks exist only for owned nodes (finalize writes dsz[u] for
    // u in [lo, hi) only), so the block offsets are a scan of the owned range
    size_t bytes = scratch_bytes;
    if (hi > lo)
        check_launch(cub::DeviceScan::ExclusiveSum(scratch, bytes, c.dsz + lo, c.doff + lo, int(hi - lo), s));
    bytes = scratch_bytes;
    check_launch(cub::DeviceScan::ExclusiveSum(scratch, bytes, c.revcnt, c.roff, int(n), s));
}

void launch_check_capacity(IterCounters* ctr, unsigned long long capacity, cudaStream_t s) {
    check_capacity_kernel<<<1, 1, 0, s>>>(ctr, capacity);
}

void launch_scatter_rev(const CandView& c, const uint32_t* active, IterCounters* ctr,
                        uint32_t max_active, uint32_t n, cudaStream_t s) {
    if (!max_active) return;
    check_launch(cudaMemsetAsync(c.rcur, 0, sizeof(uint32_t) * n, s));
    scatter_rev_kernel<<<uint32_t((size_t(max_active) * 32 + 255) / 256), 256, 0, s>>>(c, active,
                                                                                       ctr);
}

void launch_join_distances(const GraphView& g, const CandView& c, const uint32_t* active,
                           IterCounters* ctr, uint32_t max_active, cudaStream_t s) {
    if (!max_active) return;
    // resident mode when every slab of the batch's rows fits the ring with a
    // slot budget of at least one full node (2 cap column slots plus two
    // 8-paddings); otherwise pass mode
    const uint32_t n_slabs = (g.stride + kSlab - 1) / kSlab;
    const uint32_t node_slots = (2 * c.cap + 16 + 7) / 8 * 8;
    uint32_t res_slots = std::min<uint32_t>(kSlotTab, kStages * kRingRows / n_slabs / 8 * 8);
    static const bool allow_resident = [] {  // KNNG_JOIN_RESIDENT=0: pass mode always (A/B)
        const char* v = getenv("KNNG_JOIN_RESIDENT");
        return !(v && v[0] == '0');
    }();
    if (res_slots < node_slots || !allow_resident) res_slots = 0;
    // U tiles for long rows in pass mode: they cut the leftover-row padding of
    // late iterations, which binds when each tile streams many slabs (C5:
    // join 478 -> 451 ms); on short rows the extra tile phase costs more than
    // it saves (C3: 24.9 -> 26.9 ms).  KNNG_JOIN_UTILES=0 / 1 forces them
    // off / on (pass mode).
    const char* uv = getenv("KNNG_JOIN_UTILES");
    const bool utiles = res_slots == 0 && (uv ? uv[0] == '1' : g.stride >= 512);
    auto kern = utiles ? join_distances_kernel<true> : join_distances_kernel<false>;
    static int occ[kMaxDevices][2] = {};  // per device: the attribute is per device
    int& per_sm = occ[current_device()][utiles ? 1 : 0];
    if (!per_sm) {
        check_launch(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(kDistSmem)));
        int v = 0;
        check_launch(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, int(kThreads),
                                                                   kDistSmem));
        per_sm = v < 1 ? 1 : v;
    }
    uint32_t grid = device_sm_count() * uint32_t(per_sm);
    if (grid > max_active) grid = max_active;
    check_launch(cudaMemsetAsync(&ctr->work, 0, sizeof(uint32_t), s));
    kern<<<grid, kThreads, kDistSmem, s>>>(g, c, active, ctr, res_slots, -0.0f);
}

void launch_join_merge(const GraphView& g, const CandView& c, IterCounters* ctr,
                       cudaStream_t s) {
    if (g.hi <= g.lo) return;
    const uint32_t blocks = (g.hi - g.lo + kMergeWarps - 1) / kMergeWarps;
    // the hubs it left: a CTA each, blocks looping over the device-side count
    const uint32_t hub_blocks = std::min<uint32_t>(2 * device_sm_count(), (g.hi - g.lo + 1) / 2 + 1);
    if (c.det) {
        join_merge_kernel<true><<<blocks, kMergeWarps * 32, 0, s>>>(g, c, ctr, c.hubs);
        hub_merge_kernel<true><<<hub_blocks, kHubWarps * 32, 0, s>>>(g, c, ctr, c.hubs);
    } else {
        join_merge_kernel<false><<<blocks, kMergeWarps * 32, 0, s>>>(g, c, ctr, c.hubs);
        hub_merge_kernel<false><<<hub_blocks, kHubWarps * 32, 0, s>>>(g, c, ctr, c.hubs);
    }
}

// ---------------------------------------------------------------------------
// Multi-GPU: proposals for targets owned by other devices.
// ---------------------------------------------------------------------------
namespace {

// Pass 1 (count) / pass 2 (write): one warp per non-owned target t named by
// this device's lists.  The warp merges this device's proposals for t below
// t's row maximum (replicated) into an empty row and exports the entries that
// entered it, at most k per target: a proposal outside the k best distinct
// ids of this device's proposals cannot enter t's final row (SURVEY §8e
// pre-reduction; ties aside, as everywhere in the merge).  Both passes replay
// the same entries in the same order, so they agree.  Records (t, id, dist
// bits) are laid out in ascending t, hence grouped by owner device in rank
// order.
template <bool kWrite>
__global__ void __launch_bounds__(kMergeWarps * 32) export_remote_kernel(
    GraphView g, CandView c, IterCounters* ctr, uint32_t* counts, const uint64_t* offsets,
    uint32_t* records) {
    if (ctr->overflow || ctr->halt) return;
    const uint32_t lane = lane_id();
    const uint32_t t = blockIdx.x * kMergeWarps + (threadIdx.x >> 5);
    if (t >= g.n) return;
    const bool owned = t >= g.lo && t < g.hi;
    const uint32_t cnt = owned ? 0u : c.revcnt[t];
    if (!cnt) {
        if (!kWrite && lane == 0) counts[t] = 0;
        return;
    }
    const uint32_t k = g.k;
    // the row replica is not kept (partitioned shards): start from k
    // sentinels at t's row maximum (replicated) and keep the k best distinct
    // proposals below it
    const float mx = g.maxd[t];
    uint64_t key = lane < k ? pack_key(mx, 0xffffffffu) : kEmptyKey;
    uint32_t fresh = 0;  // bit i: entry i entered from this device's proposals
    float cur_max = mx;
    const uint64_t* rv = c.rev + c.roff[t];
    for (uint32_t e = 0; e < cnt; ++e) {
        const uint64_t* row = c.D + rv[e];
        const uint32_t P = uint32_t(row[0]);  // proposals kept for t in this join
        JCHECK(P <= 2 * c.cap, "export_remote row count", t, P);
        for (uint32_t q0 = 0; q0 < P; q0 += 32) {
            const uint32_t q = q0 + lane;
            const uint64_t kk = q < P ? row[1 + q] : kEmptyKey;
            uint32_t pass = __ballot_sync(0xffffffffu, q < P && key_dist(kk) < cur_max);
            while (pass) {
                const uint32_t src = __ffs(pass) - 1u;
                pass &= pass - 1u;
                const uint64_t pk = __shfl_sync(0xffffffffu, kk, src);
                const float dd = key_dist(pk);
                if (dd < cur_max && warp_try_insert(key, fresh, k, dd, key_id(pk)))
                    cur_max = key_dist(__shfl_sync(0xffffffffu, key, k - 1));
            }
        }
    }
    const uint32_t kmask = k >= 32 ? 0xffffffffu : ((1u << k) - 1u);
    fresh &= kmask;
    if (kWrite && ((fresh >> lane) & 1u)) {
        uint32_t* rec = records + 3 * (offsets[t] + __popc(fresh & ((1u << lane) - 1u)));
        rec[0] = t;
        rec[1] = key_id(key);
        rec[2] = uint32_t(key >> 32);
    }
    if (!kWrite && lane == 0) counts[t] = __popc(fresh);
}

// Received records grouped by target (counting sort), then one warp per owned
// target merges its records with try_insert semantics.
__global__ void recv_count_kernel(const uint32_t* records, uint64_t count, uint32_t* cnt) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < count) {
        JCHECK(records[3 * i] < 0x7fffffffu, "recv_count target", uint32_t(i), records[3 * i]);
        atomicAdd(cnt + records[3 * i], 1u);
    }
}

__global__ void recv_scatter_kernel(const uint32_t* records, uint64_t count, const uint32_t* off,
                                    uint32_t* cur, uint64_t* grouped) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint32_t t = records[3 * i];
    JCHECK(t < 0x7fffffffu, "recv_scatter target", uint32_t(i), t);
    const uint32_t slot = off[t] + atomicAdd(cur + t, 1u);
    grouped[slot] = pack_key(__uint_as_float(records[3 * i + 2]), records[3 * i + 1]);
}

__global__ void __launch_bounds__(kMergeWarps * 32) merge_received_kernel(
    GraphView g, const uint32_t* cnt, const uint32_t* off, const uint64_t* grouped,
    IterCounters* ctr) {
    __shared__ unsigned long long s_changes;
    if (threadIdx.x == 0) s_changes = 0;
    __syncthreads();
    const uint32_t lane = lane_id(), k = g.k;
    const uint32_t t = g.lo + blockIdx.x * kMergeWarps + (threadIdx.x >> 5);
    const uint32_t n_rec = t < g.hi ? cnt[t] : 0u;
    if (n_rec) {
        uint64_t key = lane < k ? g.keys[size_t(t) * k + lane] : kEmptyKey;
        uint32_t flags = g.flags[t];
        float cur_max = key_dist(__shfl_sync(0xffffffffu, key, k - 1));
        uint32_t inserted = 0;
        const uint64_t* recs = grouped + off[t];
        for (uint32_t r0 = 0; r0 < n_rec; r0 += 32) {
            const bool valid = r0 + lane < n_rec;
            const uint64_t rk = valid ? recs[r0 + lane] : kEmptyKey;
            uint32_t pass = __ballot_sync(0xffffffffu, valid && key_dist(rk) < cur_max);
            while (pass) {
                const uint32_t src = __ffs(pass) - 1u;
                pass &= pass - 1u;
                const uint64_t kk = __shfl_sync(0xffffffffu, rk, src);
                if (key_dist(kk) < cur_max &&
                    warp_try_insert(key, flags, k, key_dist(kk), key_id(kk))) {
                    ++inserted;
                    cur_max = key_dist(__shfl_sync(0xffffffffu, key, k - 1));
                }
            }
        }
        if (inserted) {
            if (lane < k) g.keys[size_t(t) * k + lane] = key;
            if (lane == 0) {
                g.flags[t] = flags;
                g.maxd[t] = cur_max;
                atomicAdd(&s_changes, (unsigned long long)inserted);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_changes) atomicAdd(&ctr->changes, s_changes);
}

}  // namespace

void launch_export_remote(const GraphView& g, const CandView& c, IterCounters* ctr,
                          uint32_t* counts, const uint64_t* offsets, uint32_t* records,
                          bool write, cudaStream_t s) {
    const uint32_t grid = (g.n + kMergeWarps - 1) / kMergeWarps;
    if (write)
        export_remote_kernel<true><<<grid, kMergeWarps * 32, 0, s>>>(g, c, ctr, counts, offsets,
                                                                     records);
    else
        export_remote_kernel<false><<<grid, kMergeWarps * 32, 0, s>>>(g, c, ctr, counts, offsets,
                                                                      records);
}

void launch_merge_received(const GraphView& g, const uint32_t* records, uint64_t count,
                           uint32_t* cnt, uint32_t* off, uint32_t* cur, uint64_t* grouped,
                           void* scratch, size_t scratch_bytes, IterCounters* ctr,
                           cudaStream_t s) {
    check_launch(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * g.n, s));
    check_launch(cudaMemsetAsync(cur, 0, sizeof(uint32_t) * g.n, s));
    if (count) {
        const uint32_t grid = uint32_t((count + 255) / 256);
        recv_count_kernel<<<grid, 256, 0, s>>>(records, count, cnt);
        size_t bytes = scratch_bytes;
        check_launch(cub::DeviceScan::ExclusiveSum(scratch, bytes, cnt, off, int(g.n), s));
        recv_scatter_kernel<<<grid, 256, 0, s>>>(records, count, off, cur, grouped);
    }
    if (g.hi <= g.lo || !count) return;
    merge_received_kernel<<<(g.hi - g.lo + kMergeWarps - 1) / kMergeWarps, kMergeWarps * 32, 0,
                            s>>>(g, cnt, off, grouped, ctr);
}

}  // namespace knng_cuda

#if KNNG_JOIN_STATS
// Diagnostics build only: read and clear the join counters.
extern "C" int knng_cuda_debug_join_stats(unsigned long long* out) {
    if (cudaMemcpyFromSymbol(out, knng_cuda::g_join_stats, sizeof(unsigned long long) * 8) !=
        cudaSuccess)
        return 1;
    const unsigned long long zero[8] = {};
    return cudaMemcpyToSymbol(knng_cuda::g_join_stats, zero, sizeof(zero)) != cudaSuccess;
}
#endif
