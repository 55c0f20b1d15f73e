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
// (8 x Kl bytes per row, Kl = stride / 8 rounded up to 64), adds the per-lane
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

#ifndef KNNG_U8_WARPS
#define KNNG_U8_WARPS 8
#endif
constexpr uint32_t kUWarps = KNNG_U8_WARPS;  // warps per CTA, one node each
constexpr uint32_t kUMaxM = 2 * kMaxCap;

struct U8Warp {
    int32_t nrm[kUMaxM][8];   // per-lane squared norms of the node's candidates
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

// Byte-layout of one row: lane l occupies bytes [l Kl, (l + 1) Kl), Kl a
// multiple of 64; inside a lane, each 64-byte pair of k-chunks is permuted so
// that MMA thread t's sixteen bytes (k = 4t..4t+3 and 16+4t..16+4t+3 of both
// chunks) are contiguous at 16t: one 16-byte load per row per chunk pair.  The
// permutation is the same for both MMA operands, and integer dot products do
// not depend on the order of terms (u8_pack_kernel writes it).

// All coordinates integral in [0, 255]?  flag starts at 1; any miss clears it.
// Grid-stride in chunks of 32 elements per thread; every warp re-reads the
// flag between chunks and stops once any warp has cleared it, so float data
// (the usual case: C1 / C3 / C4 / C5) is rejected after the first chunk
// instead of after a full pass over the data (C5: 2.9 -> ~0.01 ms).
__global__ void u8_check_kernel(const float* __restrict__ data, size_t count, uint32_t* flag) {
    constexpr uint32_t kPer = 32;
    const size_t span = size_t(gridDim.x) * blockDim.x;
    const size_t t = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t lane0 = t - (threadIdx.x & 31u);  // warp-uniform loop bound
    for (size_t w0 = lane0, base = t; w0 < count; w0 += span * kPer, base += span * kPer) {
        bool ok = true;
#pragma unroll 4
        for (uint32_t j = 0; j < kPer; ++j) {
            const size_t i = base + size_t(j) * span;
            if (i < count) {
                const float x = data[i];
                ok &= x >= 0.0f && x <= 255.0f && x == rintf(x);
            }
        }
        if (!__all_sync(0xffffffffu, ok)) {
            if ((threadIdx.x & 31u) == 0) atomicAnd(flag, 0u);
            return;
        }
        if (__shfl_sync(0xffffffffu, *(volatile uint32_t*)flag, 0) == 0u) return;
    }
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
    const uint32_t groups = kl / 64;  // 64-byte chunk pairs per lane
    int32_t nrm = 0;                  // lane (lane & 7)'s partial norm
    for (uint32_t w = lane; w < 8 * groups; w += 32) {
        const uint32_t l = w % 8, gi = w / 8;
        // byte p = 16 t + 8 ch + 4 h + b of the block holds k = 32 ch + 16 h + 4 t + b
        uint32_t words[16];
#pragma unroll
        for (uint32_t wi = 0; wi < 16; ++wi) {
            const uint32_t t = wi / 4, ch = (wi % 4) / 2, h = wi % 2;
            uint32_t v = 0;
#pragma unroll
            for (uint32_t b = 0; b < 4; ++b) {
                const uint32_t e = 8 * (gi * 64 + 32 * ch + 16 * h + 4 * t + b) + l;
                const uint32_t xv = e < stride ? uint32_t(x[e]) : 0u;
                v |= xv << (8 * b);
                nrm += int32_t(xv * xv);
            }
            words[wi] = v;
        }
        uint4* dst = reinterpret_cast<uint4*>(out + l * kl + gi * 64);
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q)
            dst[q] = make_uint4(words[4 * q], words[4 * q + 1], words[4 * q + 2], words[4 * q + 3]);
    }
    // lanes congruent mod 8 hold the same reference lane
    nrm += __shfl_xor_sync(0xffffffffu, nrm, 8);
    nrm += __shfl_xor_sync(0xffffffffu, nrm, 16);
    if (lane < 8) lnorm[size_t(row) * 8 + lane] = nrm;
}

#ifndef KNNG_U8_NB
#define KNNG_U8_NB 1  // 1 measured 10% faster than 2 and 4 (C2 join per build)
#endif
constexpr uint32_t kUNB = KNNG_U8_NB;  // column blocks per pass
// fragment loads from the byte copy: 0 read-only path (__ldg), 1 L2 only
// (__ldcg), 2 read-only without L1 allocation (A/B builds: scripts/build_variants.py)
#ifndef KNNG_U8_LD
#define KNNG_U8_LD 0
#endif
__device__ __forceinline__ uint4 ld_frag(const uint8_t* p) {
#if KNNG_U8_LD == 1
    return __ldcg(reinterpret_cast<const uint4*>(p));
#elif KNNG_U8_LD == 2
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
#else
    return __ldg(reinterpret_cast<const uint4*>(p));
#endif
}
#ifndef KNNG_U8_MINB
#define KNNG_U8_MINB 2  // CTAs per SM the register budget is sized for
#endif

// One 16-row block (mi) of new candidates against kUNB 8-column blocks from
// njb: per reference lane l, the C k-chunks' fragments are all loaded before
// the MMAs (the byte rows come from L2: latency, not bandwidth, bounds a
// dependent load -> MMA chain), then the lane sums enter the FP32 tree; the
// pairs' proposals are written at the end.
//
// SW (swapped, nodes with nn <= 8): the 16 MMA rows run over candidates j
// (block mi of all m) and the 8 columns over the new candidates i (block 0),
// so a short new list fills 8 rather than 16 MMA rows: half the tiles.
template <uint32_t C2, bool SW = false>
__device__ __forceinline__ void tile_pairs(U8Warp& W, const uint8_t* __restrict__ packed,
                                           uint32_t kl, uint32_t mi, uint32_t njb, uint32_t nn,
                                           uint32_t m, uint32_t nnj, int filter, uint64_t* D) {
    // C2 = 64-byte chunk pairs per lane (Kl / 64)
    const uint32_t lane = threadIdx.x & 31u, gq = lane >> 2, t = lane & 3u;
    const size_t row_bytes = size_t(8) * kl;
    const uint32_t ra0 = 16 * mi + gq, ra1 = ra0 + 8;
    const uint8_t* pa0 = packed + size_t(W.rid[ra0]) * row_bytes + 16 * t;
    const uint8_t* pa1 = packed + size_t(W.rid[ra1]) * row_bytes + 16 * t;
    const uint8_t* pb[kUNB];
    uint32_t cb[kUNB];
    bool live[kUNB];
#pragma unroll
    for (uint32_t q = 0; q < kUNB; ++q) {
        live[q] = njb + q < nnj;
        const uint32_t col = min(8 * (njb + q) + gq, kUMaxM - 1);
        cb[q] = min(8 * (njb + q) + 2 * t, kUMaxM - 2);
        pb[q] = packed + size_t(W.rid[live[q] ? col : 0]) * row_bytes + 16 * t;
    }
    // tree partials of the kUNB x 4 C elements (see the lane schedule below)
    float part[kUNB][4][3];
#pragma unroll
    for (uint32_t l = 0; l < 8; ++l) {
        uint4 A0[C2], A1[C2], B[kUNB][C2];
#pragma unroll
        for (uint32_t g2 = 0; g2 < C2; ++g2) {
            const size_t o = size_t(l) * kl + 64 * g2;
            A0[g2] = ld_frag(pa0 + o);
            A1[g2] = ld_frag(pa1 + o);
#pragma unroll
            for (uint32_t q = 0; q < kUNB; ++q) B[q][g2] = ld_frag(pb[q] + o);
        }
        int acc[kUNB][4];
#pragma unroll
        for (uint32_t q = 0; q < kUNB; ++q)
#pragma unroll
            for (uint32_t r = 0; r < 4; ++r) acc[q][r] = 0;
#pragma unroll
        for (uint32_t g2 = 0; g2 < C2; ++g2)
#pragma unroll
            for (uint32_t q = 0; q < kUNB; ++q) {
                mma_u8(acc[q], A0[g2].x, A1[g2].x, A0[g2].y, A1[g2].y, B[q][g2].x, B[q][g2].y);
                mma_u8(acc[q], A0[g2].z, A1[g2].z, A0[g2].w, A1[g2].w, B[q][g2].z, B[q][g2].w);
            }
        // lane sums (exact integers < 2^24) into the reference's tree
        // ((0+1)+(2+3))+((4+5)+(6+7)): p0 holds s0 / s01 / s4 / s45, p1 s2 / s6,
        // p2 s0123; after lane 7 p0 is the distance
        const int32_t a_n0 = W.nrm[ra0][l], a_n1 = W.nrm[ra1][l];
#pragma unroll
        for (uint32_t q = 0; q < kUNB; ++q) {
            const int32_t b_n0 = W.nrm[cb[q]][l], b_n1 = W.nrm[cb[q] + 1][l];
#pragma unroll
            for (uint32_t r = 0; r < 4; ++r) {
                const int32_t an = r < 2 ? a_n0 : a_n1;
                const int32_t bn = (r & 1u) ? b_n1 : b_n0;
                const float sl = float(an + bn - 2 * acc[q][r]);
                float* p = part[q][r];
                if (l == 0 || l == 4)
                    p[0] = sl;
                else if (l == 2 || l == 6)
                    p[1] = sl;
                else if (l == 1 || l == 5)
                    p[0] = __fadd_rn(p[0], sl);
                else if (l == 3)
                    p[2] = __fadd_rn(p[0], __fadd_rn(p[1], sl));
                else
                    p[0] = __fadd_rn(p[2], __fadd_rn(p[0], __fadd_rn(p[1], sl)));
            }
        }
    }
#pragma unroll
    for (uint32_t q = 0; q < kUNB; ++q) {
        if (!live[q]) continue;
#pragma unroll
        for (uint32_t r = 0; r < 4; ++r) {
            const uint32_t ra = 16 * mi + gq + 8 * (r >> 1);
            const uint32_t cb_ = 8 * (njb + q) + 2 * t + (r & 1u);
            const uint32_t i = SW ? cb_ : ra, j = SW ? ra : cb_;
            if (i >= nn || j >= m || (j < nn && j <= i)) continue;
            const uint32_t id_i = W.rid[i], id_j = W.rid[j];
            // an id listed twice pairs with itself: try_insert ignores self
            // (graph.hpp:116-129)
            if (filter && id_i == id_j) continue;
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

template <uint32_t C>
__global__ void __launch_bounds__(kUWarps * 32, KNNG_U8_MINB) join_u8_kernel(GraphView g, CandView c,
                                                               IterCounters* ctr,
                                                               const uint8_t* __restrict__ packed,
                                                               const int32_t* __restrict__ lnorm,
                                                               uint32_t kl, uint32_t heavy_nn,
                                                               int no_swap) {
    __shared__ U8Warp shw[kUWarps];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    U8Warp& W = shw[warp];
    if (ctr->overflow || ctr->halt) return;
    const uint32_t n_active = ctr->active, cap = c.cap;
    for (;;) {
        uint32_t a = 0;
        if (lane == 0) a = atomicAdd(&ctr->work, 1u);
        a = __shfl_sync(0xffffffffu, a, 0);
        if (a >= n_active) break;
        const uint4 rec = c.arec[a];
        const uint32_t u = rec.x, nn = rec.y & 0xffffu, no = rec.y >> 16, m = nn + no;
        if (nn > heavy_nn) continue;  // join_u8_staged_kernel's node
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
        // the lane norms (32 bytes each, 4 threads per row) of the rows the
        // tiles read: the candidates and the padding of the last blocks
        const bool swapped = nn <= 8 && !no_swap;
        const uint32_t rows =
            swapped ? 16 * ((m + 15) / 16) : max(16 * ((nn + 15) / 16), 8 * ((m + 7) / 8));
        for (uint32_t q = lane; q < 4 * rows; q += 32) {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(lnorm + size_t(W.rid[q >> 2]) * 8) +
                                  (q & 3u));
            W.nrm[q >> 2][2 * (q & 3u)] = int32_t(v.x);
            W.nrm[q >> 2][2 * (q & 3u) + 1] = int32_t(v.y);
        }
        __syncwarp();
        const uint32_t nmi = (nn + 15) / 16, nnj = (m + 7) / 8;
        if (swapped) {
            for (uint32_t mj = 0; mj < (m + 15) / 16; ++mj)
                tile_pairs<C, true>(W, packed, kl, mj, 0, nn, m, 1, c.filter, D);
        } else {
            for (uint32_t mi = 0; mi < nmi; ++mi)
                // column blocks left of the diagonal block hold only pairs j <= i
                for (uint32_t njb = 2 * mi; njb < nnj; njb += kUNB)
                    tile_pairs<C>(W, packed, kl, mi, njb, nn, m, nnj, c.filter, D);
        }
        __syncwarp();
        for (uint32_t x = lane; x < m; x += 32) D[u8_prow(x, nn, m)] = W.rowcnt[x];
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Staged variant: one CTA per active node, the node's byte rows and lane
// norms copied once into shared memory (16-byte cp.async, L2 -> SMEM), then
// the CTA's warps split the node's (16-row block, 2 column blocks) tiles.  The
// warp-per-node kernel above reads every fragment from L2 once per tile that
// uses it (A rows once per column-block pair, B rows once per row block); here
// each row crosses L2 once per node.  Two CTAs per SM: one stages while the
// other computes; the next node's record, ids and row maxima are loaded into
// registers while the current node's copies are in flight.  Arithmetic,
// tree order and proposal epilogue are those of tile_pairs (bit-identical).
// Nodes with more than heavy_nn new candidates (KNNG_U8_HEAVY, default 16)
// come here, claimed 32 active indices at a time; the rest stay with the
// warp-per-node kernel, which skips them.
//
// Measured slower on B200 and kept opt-in (KNNG_U8_STAGED=1): C2 join 6.0 ->
// 7.4 ms per build (heavy > 16), 8.3 ms (> 8), 10.3 ms (every node);
// iteration 1 1.63 -> 2.09 ms.  ncu (profiles/round1_ncu_join_u8_staged_c2.json):
// 57% more instructions than the warp kernel (swizzled shared addressing, no
// immediate offsets), issue active 36%, the top stall the node barriers: with
// 7 tile units per iteration-1 node and 8 warps, each warp runs one
// dependent load -> MMA chain per node, and two CTAs per SM do not hide the
// staging round trip.
//
// Shared rows are 8 Kl bytes with no padding; the 16-byte chunks of odd rows
// are XOR-swizzled by 64 bytes, so the two rows a quarter-warp's 16-byte
// fragment loads touch (gq, gq + 1) fall in different bank halves.
constexpr uint32_t kSWarps = 8;

__device__ __forceinline__ void cp_async16_u8(void* smem_dst, const void* gmem_src) {
    const uint32_t dst = uint32_t(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(gmem_src));
}

struct U8Stage {
    const uint8_t* rows;  // m x 8 Kl bytes, swizzled
    const int32_t* nrm;   // m x 8
    const uint32_t* rid;  // m
    const float* rmx;     // m
    uint32_t* rowcnt;     // m
};

template <uint32_t C2>
__device__ __forceinline__ void tile_pairs_staged(const U8Stage& S, uint32_t mi, uint32_t njb,
                                                  uint32_t nn, uint32_t m, uint32_t nnj, int filter,
                                                  uint64_t* D) {
    constexpr uint32_t kl = 64 * C2, RB = 8 * kl;
    const uint32_t lane = threadIdx.x & 31u, gq = lane >> 2, t = lane & 3u;
    // rows past the node's list (padding of the last 16 / 8 blocks) read row 0
    auto srow = [&](uint32_t r) { return r < m ? r : 0u; };
    const uint32_t ra0 = srow(16 * mi + gq), ra1 = srow(16 * mi + gq + 8);
    // byte offsets of this thread's fragment rows; the swizzle of a row's
    // chunk offset o is o ^ ((row & 1) << 6)
    const uint32_t oa0 = ra0 * RB, oa1 = ra1 * RB, sa0 = (ra0 & 1u) << 6, sa1 = (ra1 & 1u) << 6;
    uint32_t ob[kUNB], sb[kUNB], cb0[kUNB], cb1[kUNB];
    bool live[kUNB];
#pragma unroll
    for (uint32_t q = 0; q < kUNB; ++q) {
        live[q] = njb + q < nnj;
        const uint32_t col = srow(8 * (njb + q) + gq);
        ob[q] = col * RB;
        sb[q] = (col & 1u) << 6;
        cb0[q] = srow(8 * (njb + q) + 2 * t) * 8;
        cb1[q] = srow(8 * (njb + q) + 2 * t + 1) * 8;
    }
    float part[kUNB][4][3];
#pragma unroll
    for (uint32_t l = 0; l < 8; ++l) {
        uint4 A0[C2], A1[C2], B[kUNB][C2];
#pragma unroll
        for (uint32_t g2 = 0; g2 < C2; ++g2) {
            const uint32_t o = l * kl + 64 * g2 + 16 * t;
            A0[g2] = *reinterpret_cast<const uint4*>(S.rows + (oa0 + (o ^ sa0)));
            A1[g2] = *reinterpret_cast<const uint4*>(S.rows + (oa1 + (o ^ sa1)));
#pragma unroll
            for (uint32_t q = 0; q < kUNB; ++q)
                B[q][g2] = *reinterpret_cast<const uint4*>(S.rows + (ob[q] + (o ^ sb[q])));
        }
        int acc[kUNB][4];
#pragma unroll
        for (uint32_t q = 0; q < kUNB; ++q)
#pragma unroll
            for (uint32_t r = 0; r < 4; ++r) acc[q][r] = 0;
#pragma unroll
        for (uint32_t g2 = 0; g2 < C2; ++g2)
#pragma unroll
            for (uint32_t q = 0; q < kUNB; ++q) {
                mma_u8(acc[q], A0[g2].x, A1[g2].x, A0[g2].y, A1[g2].y, B[q][g2].x, B[q][g2].y);
                mma_u8(acc[q], A0[g2].z, A1[g2].z, A0[g2].w, A1[g2].w, B[q][g2].z, B[q][g2].w);
            }
        // the reference's tree, as in tile_pairs
        const int32_t a_n0 = S.nrm[ra0 * 8 + l], a_n1 = S.nrm[ra1 * 8 + l];
#pragma unroll
        for (uint32_t q = 0; q < kUNB; ++q) {
            const int32_t b_n0 = S.nrm[cb0[q] + l], b_n1 = S.nrm[cb1[q] + l];
#pragma unroll
            for (uint32_t r = 0; r < 4; ++r) {
                const int32_t an = r < 2 ? a_n0 : a_n1;
                const int32_t bn = (r & 1u) ? b_n1 : b_n0;
                const float sl = float(an + bn - 2 * acc[q][r]);
                float* p = part[q][r];
                if (l == 0 || l == 4)
                    p[0] = sl;
                else if (l == 2 || l == 6)
                    p[1] = sl;
                else if (l == 1 || l == 5)
                    p[0] = __fadd_rn(p[0], sl);
                else if (l == 3)
                    p[2] = __fadd_rn(p[0], __fadd_rn(p[1], sl));
                else
                    p[0] = __fadd_rn(p[2], __fadd_rn(p[0], __fadd_rn(p[1], sl)));
            }
        }
    }
#pragma unroll
    for (uint32_t q = 0; q < kUNB; ++q) {
        if (!live[q]) continue;
#pragma unroll
        for (uint32_t r = 0; r < 4; ++r) {
            const uint32_t i = 16 * mi + gq + 8 * (r >> 1);
            const uint32_t j = 8 * (njb + q) + 2 * t + (r & 1u);
            if (i >= nn || j >= m || (j < nn && j <= i)) continue;
            const uint32_t id_i = S.rid[i], id_j = S.rid[j];
            if (filter && id_i == id_j) continue;  // try_insert ignores self
            const float dist = part[q][r][0];
            if (dist < S.rmx[i]) {
                const uint32_t pos = atomicAdd(&S.rowcnt[i], 1u);
                D[u8_prow(i, nn, m) + 1 + pos] = pack_key(dist, id_j);
            }
            if (dist < S.rmx[j]) {
                const uint32_t pos = atomicAdd(&S.rowcnt[j], 1u);
                D[u8_prow(j, nn, m) + 1 + pos] = pack_key(dist, id_i);
            }
        }
    }
}

__host__ __device__ constexpr size_t u8_staged_smem(uint32_t C2, uint32_t mmax) {
    return size_t(mmax) * (512u * C2 + 32u + 12u);
}

template <uint32_t C2>
__global__ void __launch_bounds__(kSWarps * 32, 2)
    join_u8_staged_kernel(GraphView g, CandView c, IterCounters* ctr,
                          const uint8_t* __restrict__ packed, const int32_t* __restrict__ lnorm,
                          uint32_t heavy_nn) {
    constexpr uint32_t RB = 512 * C2, CH = RB / 16;  // row bytes, 16-byte chunks per row
    extern __shared__ __align__(16) uint8_t u8s[];
    const uint32_t cap = c.cap, mmax = 2 * cap, tid = threadIdx.x, warp = tid >> 5;
    U8Stage S;
    uint8_t* rows = u8s;
    int32_t* nrm = reinterpret_cast<int32_t*>(u8s + size_t(mmax) * RB);
    uint32_t* rid = reinterpret_cast<uint32_t*>(nrm + size_t(mmax) * 8);
    float* rmx = reinterpret_cast<float*>(rid + mmax);
    uint32_t* rowcnt = reinterpret_cast<uint32_t*>(rmx + mmax);
    S.rows = rows;
    S.nrm = nrm;
    S.rid = rid;
    S.rmx = rmx;
    S.rowcnt = rowcnt;
    if (ctr->overflow || ctr->halt) return;
    const uint32_t n_active = ctr->active, lane = tid & 31u;
    const float inf = __int_as_float(0x7f800000);
    // work queue: warp 0 claims 32 active indices at a time and keeps the
    // records of the heavy ones (nn > heavy_nn); the rest are the warp-per-node
    // kernel's
    __shared__ uint4 q_rec[32];
    __shared__ uint32_t q_n;
    auto refill = [&]() -> uint32_t {
        for (;;) {
            if (warp == 0) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(&ctr->work2, 32u);
                base = __shfl_sync(0xffffffffu, base, 0);
                const uint32_t idx = base + lane;
                uint4 r = make_uint4(0, 0, 0, 0);
                if (idx < n_active) r = c.arec[idx];
                const bool heavy = idx < n_active && (r.y & 0xffffu) > heavy_nn;
                const uint32_t mask = __ballot_sync(0xffffffffu, heavy);
                if (heavy) q_rec[__popc(mask & ((1u << lane) - 1u))] = r;
                if (lane == 0) q_n = base >= n_active ? 0xffffffffu : __popc(mask);
            }
            __syncthreads();
            const uint32_t qn = q_n;
            if (qn) return qn == 0xffffffffu ? 0u : qn;
            __syncthreads();  // q_n is rewritten by the next claim
        }
    };
    // this thread's candidate (x = tid) of a node: id and row maximum
    auto fetch = [&](const uint4& rec, uint32_t& id, float& mx) {
        const uint32_t nn = rec.y & 0xffffu, m = nn + (rec.y >> 16);
        if (tid < m) {
            const size_t pos = size_t(rec.x) * 2 * cap + (tid < nn ? tid : cap + tid - nn);
            id = c.ids[pos];
            mx = c.filter ? c.cmax[pos] : inf;
        }
    };
    uint32_t qn = refill(), qi = 0;
    if (!qn) return;
    uint4 rec = q_rec[0];
    uint32_t pid = 0;
    float pmx = inf;
    fetch(rec, pid, pmx);
    for (;;) {
        const uint32_t nn = rec.y & 0xffffu, m = nn + (rec.y >> 16);
        uint64_t* const D = c.D + (uint64_t(rec.z) | (uint64_t(rec.w) << 32));
        if (tid < m) {
            rid[tid] = pid;
            rmx[tid] = pmx;
            rowcnt[tid] = 0;
        }
        __syncthreads();
        for (uint32_t q = tid; q < m * CH; q += kSWarps * 32) {
            const uint32_t x = q / CH, ch = q % CH;
            cp_async16_u8(rows + size_t(x) * RB + ((16 * ch) ^ ((x & 1u) << 6)),
                          packed + size_t(rid[x]) * RB + 16 * ch);
        }
        for (uint32_t q = tid; q < 2 * m; q += kSWarps * 32)
            cp_async16_u8(nrm + 4 * q, lnorm + size_t(rid[q >> 1]) * 8 + 4 * (q & 1u));
        asm volatile("cp.async.commit_group;\n" ::);
        // the next queued node's candidates load while the copies are in flight
        uint4 rec_next = rec;
        if (qi + 1 < qn) {
            rec_next = q_rec[qi + 1];
            fetch(rec_next, pid, pmx);
        }
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();
        const uint32_t nmi = (nn + 15) / 16, nnj = (m + 7) / 8;
        uint32_t unit = 0;
        for (uint32_t mi = 0; mi < nmi; ++mi)
            for (uint32_t njb = 2 * mi; njb < nnj; njb += kUNB, ++unit)
                if (unit % kSWarps == warp) tile_pairs_staged<C2>(S, mi, njb, nn, m, nnj, c.filter, D);
        __syncthreads();
        if (tid < m) D[u8_prow(tid, nn, m)] = rowcnt[tid];
        if (++qi < qn) {
            rec = rec_next;
        } else {
            qn = refill();
            if (!qn) break;
            qi = 0;
            rec = q_rec[0];
            fetch(rec, pid, pmx);
        }
    }
}

}  // namespace

uint32_t u8_lane_bytes(uint32_t stride) { return (stride / 8 + 63) / 64 * 64; }

bool u8_eligible(const float* data, uint32_t n, uint32_t stride, uint32_t* d_flag,
                 cudaStream_t s) {
    // lane sums stay below 2^24: (stride / 8) * 255^2 < 2^24
    if (stride / 8 > 258) return false;
    const uint32_t one = 1;
    check_launch(cudaMemcpyAsync(d_flag, &one, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    u8_check_kernel<<<4 * device_sm_count(), 256, 0, s>>>(data, size_t(n) * stride, d_flag);
    uint32_t h = 0;
    check_launch(cudaMemcpyAsync(&h, d_flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    check_launch(cudaStreamSynchronize(s), "byte-valued data check");
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
    const uint32_t kl = u8_lane_bytes(g.stride);
    // staged variant (opt-in, KNNG_U8_STAGED=1; measured slower, see the
    // comment above join_u8_staged_kernel) when two CTAs' node stages fit an
    // SM's shared memory (C2: 100 rows x 1 KB)
    const char* senv = getenv("KNNG_U8_STAGED");
    const bool staged_env = senv && senv[0] == '1';
    const uint32_t c2 = kl / 64;
    const size_t ssm = u8_staged_smem(c2, 2 * c.cap);
    uint32_t heavy_nn = 0xffffffffu;  // nodes with nn > heavy_nn take the staged kernel
    if (staged_env && c2 <= 2 && 2 * (ssm + 1024) <= 233472) {
        const char* hv = getenv("KNNG_U8_HEAVY");
        heavy_nn = hv ? uint32_t(atoi(hv)) : 16u;
        uint32_t grid = 2 * device_sm_count();
        if (grid > max_active) grid = max_active;
        check_launch(cudaMemsetAsync(&ctr->work2, 0, sizeof(uint32_t), s));
        if (c2 == 1) {
            cudaFuncSetAttribute(join_u8_staged_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(ssm));
            join_u8_staged_kernel<1><<<grid, kSWarps * 32, ssm, s>>>(g, c, ctr, packed, lnorm,
                                                                      heavy_nn);
        } else {
            cudaFuncSetAttribute(join_u8_staged_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(ssm));
            join_u8_staged_kernel<2><<<grid, kSWarps * 32, ssm, s>>>(g, c, ctr, packed, lnorm,
                                                                      heavy_nn);
        }
    }
    // nodes with nn <= 8 take the swapped tile shape; KNNG_U8_SWAP=0 turns it off (A/B)
    const char* wenv = getenv("KNNG_U8_SWAP");
    const int no_swap = (wenv && wenv[0] == '0') ? 1 : 0;
    static int occ[kMaxDevices] = {};
    int& per_sm = occ[current_device()];
    if (!per_sm) {
        int v = 0;
        check_launch(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, join_u8_kernel<2>,
                                                                   int(kUWarps * 32), 0));
        per_sm = v < 1 ? 1 : v;
    }
    uint32_t grid = device_sm_count() * uint32_t(per_sm);
    const uint32_t need = (max_active + kUWarps - 1) / kUWarps;
    if (grid > need) grid = need;
    check_launch(cudaMemsetAsync(&ctr->work, 0, sizeof(uint32_t), s));
#define KNNG_U8_CASE(CH)                                                                   \
    case CH:                                                                               \
        join_u8_kernel<CH><<<grid, kUWarps * 32, 0, s>>>(g, c, ctr, packed, lnorm, kl, heavy_nn, \
                                                          no_swap);                         \
        break;
    switch (kl / 64) {
        KNNG_U8_CASE(1)
        KNNG_U8_CASE(2)
        KNNG_U8_CASE(3)
        KNNG_U8_CASE(4)
        default:
            join_u8_kernel<5><<<grid, kUWarps * 32, 0, s>>>(g, c, ctr, packed, lnorm, kl, heavy_nn,
                                                            no_swap);
    }
#undef KNNG_U8_CASE
}

}  // namespace knng_cuda
