// The local-join distance stage for long rows, loading candidate rows straight
// from HBM/L2 into registers (no shared-memory staging, no CTA barriers).
//
// Same contract as join_distances_kernel (join.cu): for every active node u it
// evaluates the C(nn,2) new x new and nn*no new x old pairs of compute_step
// (reference descent.hpp:82-153) with the reference's lane-split arithmetic,
// bit for bit (distance.hpp:29-190: eight strided lanes, tree reduction,
// FMA-contracted inside full 5x5 / triangular tiles, unfused elsewhere), and
// writes every pair that beats an endpoint's iteration-start row maximum into
// u's proposal block (prefilter of descent.hpp:97-102,134-147).
//
// Differences from join.cu, all in scheduling and data movement:
//  * Lane-major copy of the data (gl_pack_kernel): in every 16-float
//    half-slab h of a row, position 2 l + c holds element 16 h + 8 c + l, so
//    one 8-byte load by thread l8 of a group returns its reference lane's
//    chunks 2h and 2h+1, in order; eight threads read one 64-byte run.  Rows
//    are zero-padded to a multiple of 16 floats (0 - 0 adds +0 exactly).
//  * Pair tiles match the reference's fused/unfused split without padding
//    the leftover rows to 8: fused pairs run in 8 x 8 tiles (A = 8 fused new
//    rows, B = 8 fused columns), unfused pairs in 4 x 16 tiles whose short
//    side is at most 4 leftover candidates — the nn % 5 leftover new rows
//    against every later column (U2), or the <= 8 leftover columns against
//    16 fused rows (U1).  A late-iteration node with nn = 4, no = 26 needs
//    two 4 x 16 tiles (110 of 128 slots live) instead of five 8 x 8.
//  * Warps are independent: a warp claims four active nodes; nodes with
//    nn <= 4 (only U2 tiles) go one per 8-thread group, larger nodes are
//    processed by the whole warp, tile by tile.  Candidate ids, row maxima
//    and proposal-row counters live in the warp's slice of shared memory.
//  * Every load is double-buffered one half-slab ahead in registers.
#include <cstdio>

#include "kernels.cuh"
#include "tile_math.cuh"

namespace knng_cuda {

namespace {

#ifndef KNNG_GL_MINBLOCKS
#define KNNG_GL_MINBLOCKS 3
#endif
#ifndef KNNG_GL_DB
#define KNNG_GL_DB 0  // 1: loads double-buffered in registers; 0: one buffer + L2 prefetch
#endif
constexpr uint32_t kGlThreads = 128;
constexpr uint32_t kGlWarps = kGlThreads / 32;
constexpr uint32_t kGlMaxM = 2 * kMaxCap;

struct GlNode {
    uint32_t id[kGlMaxM];   // candidate index -> data row id (new first, then old)
    float mx[kGlMaxM];      // its iteration-start row maximum (+inf: unfiltered)
    uint32_t cnt[kGlMaxM];  // proposals kept in its row of the node's block
};

struct GlShared {
    GlNode node[kGlWarps][4];
};

// Per-node tile geometry.  Candidate index spaces: new 0..nn-1, old nn..m-1.
//  fused rows F_r = new [0, fn), fn = nn - nn % 5; fused columns
//  F_c = new [0, fn) ++ old [0, fo), fo = no - no % 5 (column f -> candidate
//  f < fn ? f : nn + f - fn); leftover columns U_c = new [fn, nn) ++ old
//  [fo, no) (uc <= 8); leftover rows U_r = new [fn, nn) (<= 4).
//  F  tiles (8 x 8, fused):  rows 8rb.., columns 8cb.., cb >= rb
//  U1 tiles (4 x 16):        short = 4 of U_c, long = 16 of F_r (all pairs valid)
//  U2 tiles (4 x 16):        short = U_r, long = 16 of U_r ++ old (new-new: j > i)
struct GlGeom {
    uint32_t nn, no, m, fn, fo, cf, uc, l2, RB, CB, nF, q16, nU1, nU2;
    __device__ __forceinline__ bool diag_live(uint32_t rb) const {
        return min(8 * rb + 8, cf) - 1 > 8 * rb;
    }
    __device__ __forceinline__ void set(uint32_t nn_, uint32_t no_) {
        nn = nn_;
        no = no_;
        m = nn + no;
        fn = nn - nn % 5;
        fo = no - no % 5;
        cf = fn + fo;
        uc = (nn - fn) + (no - fo);
        l2 = nn > fn ? (nn - fn) + no : 0u;
        RB = (fn + 7) / 8;
        CB = (cf + 7) / 8;
        nF = 0;
        for (uint32_t rb = 0; rb < RB; ++rb) nF += CB - rb - (diag_live(rb) ? 0u : 1u);
        q16 = (fn + 15) / 16;
        nU1 = fn && uc ? ((uc + 3) / 4) * q16 : 0u;
        nU2 = (l2 + 15) / 16;
    }
    __device__ __forceinline__ uint32_t fcol(uint32_t f) const { return f < fn ? f : nn + f - fn; }
    __device__ __forceinline__ uint32_t ucol(uint32_t u) const {
        return u < nn - fn ? fn + u : nn + fo + (u - (nn - fn));
    }
    __device__ __forceinline__ uint32_t l2col(uint32_t v) const {
        return v < nn - fn ? fn + v : nn + (v - (nn - fn));
    }
    // F tile t -> (rb, cb)
    __device__ __forceinline__ void ftile(uint32_t t, uint32_t& rb, uint32_t& cb) const {
        rb = 0;
        for (;;) {
            const uint32_t first = rb + (diag_live(rb) ? 0u : 1u);
            const uint32_t cnt = CB - first;
            if (t < cnt) {
                cb = first + t;
                return;
            }
            t -= cnt;
            ++rb;
        }
    }
};

constexpr uint32_t kNone = 0xffffffffu;

// One pair tile of R x C rows (R * C = 64) over all half-slabs: thread l8 of
// the group accumulates reference lane l8 of every pair; acc[x * C/2 + j]
// holds pairs (x, 2j) and (x, 2j + 1).  ra / rc: the rows' first half-slab
// index (row * H); padding slots name the all-zero row n of the copy.
template <uint32_t R, uint32_t C, bool kFused>
__device__ __forceinline__ void gl_tile(const char* __restrict__ base, uint32_t H, const uint32_t (&ra)[R],
                                        const uint32_t (&rc)[C], float2 mz,
                                        float2 (&acc)[32]) {
    static_assert(R * C == 64, "64 pairs per tile");
    const float2 minus_one = make_float2(-1.0f, -1.0f);
    float2 a0[R], b0[C], a1[R], b1[C];
    auto load = [&](uint32_t h, float2 (&a)[R], float2 (&b)[C]) {
#pragma unroll
        for (uint32_t x = 0; x < R; ++x)
            a[x] = __ldg(reinterpret_cast<const float2*>(base + uint64_t(ra[x] + h) * 64));
#pragma unroll
        for (uint32_t y = 0; y < C; ++y)
            b[y] = __ldg(reinterpret_cast<const float2*>(base + uint64_t(rc[y] + h) * 64));
    };
    auto compute = [&](const float2 (&a)[R], const float2 (&b)[C]) {
#pragma unroll
        for (uint32_t c = 0; c < 2; ++c) {
#pragma unroll
            for (uint32_t x = 0; x < R; ++x) {
                const float av = c ? a[x].y : a[x].x;
                const float2 ax = make_float2(av, av);
#pragma unroll
                for (uint32_t j = 0; j < C / 2; ++j) {
                    const float2 bb = c ? make_float2(b[2 * j].y, b[2 * j + 1].y)
                                        : make_float2(b[2 * j].x, b[2 * j + 1].x);
                    const float2 diff = __ffma2_rn(bb, minus_one, ax);  // a - b, exact
                    float2& s = acc[x * (C / 2) + j];
                    if (kFused)
                        s = __ffma2_rn(diff, diff, s);
                    else
                        s = __fadd2_rn(s, __ffma2_rn(diff, diff, mz));  // rounded square, then add
                }
            }
        }
    };
#pragma unroll
    for (uint32_t p = 0; p < 32; ++p) acc[p] = make_float2(0.0f, 0.0f);
#if KNNG_GL_DB
    load(0, a0, b0);
    for (uint32_t h = 0; h < H; h += 2) {
        if (h + 1 < H) load(h + 1, a1, b1);
        compute(a0, b0);
        if (h + 1 >= H) break;
        if (h + 2 < H) load(h + 2, a0, b0);
        compute(a1, b1);
    }
#else
    // one buffer; the half-slab after next is prefetched into L2
    (void)a1;
    (void)b1;
    auto prefetch = [&](uint32_t h) {
#pragma unroll
        for (uint32_t x = 0; x < R; ++x)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(base + uint64_t(ra[x] + h) * 64));
#pragma unroll
        for (uint32_t y = 0; y < C; ++y)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(base + uint64_t(rc[y] + h) * 64));
    };
    if (H > 1) prefetch(1);
    for (uint32_t h = 0; h < H; ++h) {
        load(h, a0, b0);
        if (h + 2 < H) prefetch(h + 2);
        compute(a0, b0);
    }
#endif
}

__device__ __forceinline__ void gl_propose(const CandView& c, GlNode& nd, uint64_t* D,
                                           uint32_t nn, uint32_t m, uint32_t p, uint32_t q,
                                           float dist) {
    const uint32_t ip = nd.id[p], iq = nd.id[q];
    // an id listed twice pairs with itself: try_insert ignores self
    // (graph.hpp:116-129); the unfiltered entry keeps every pair
    if (c.filter && ip == iq) return;
    if (dist < nd.mx[p]) {
        const uint32_t pos = atomicAdd(&nd.cnt[p], 1u);
        D[prow(p, nn, m) + 1 + pos] = pack_key(dist, iq);
    }
    if (dist < nd.mx[q]) {
        const uint32_t pos = atomicAdd(&nd.cnt[q], 1u);
        D[prow(q, nn, m) + 1 + pos] = pack_key(dist, ip);
    }
}

// One F tile (kF) or U tile of node nd, or nothing (t == kNone: an idle group
// still runs the arithmetic on zero rows, keeping the warp converged).
template <bool kF>
__device__ __forceinline__ void gl_run_tile(const CandView& c, GlNode& nd, const GlGeom& ng,
                                            uint64_t doff, uint32_t t, const char* base,
                                            uint32_t zero_row, uint32_t H, uint32_t l8,
                                            float2 mz) {
    constexpr uint32_t R = kF ? 8 : 4, C = kF ? 8 : 16;
    // the tile's short (A) and long (B) sides as candidate indices:
    //   F:  A x -> 8 rb + x (< fn),        B y -> fcol(8 cb + y) (< cf)
    //   U1: A x -> ucol(4 rb + x) (< uc),  B y -> 16 cb + y (< fn)
    //   U2: A x -> fn + x (< nn),          B y -> l2col(16 cb + y) (< l2)
    uint32_t kind = 0, rb = 0, cb = 0;  // kind: 0 = F, 1 = U1, 2 = U2
    if (t != kNone) {
        if (kF) {
            ng.ftile(t, rb, cb);
        } else if (t < ng.nU1) {
            kind = 1;
            rb = t / ng.q16;
            cb = t % ng.q16;
        } else {
            kind = 2;
            cb = t - ng.nU1;
        }
    }
    auto a_idx = [&](uint32_t x) -> uint32_t {
        if (t == kNone) return kNone;
        if (kind == 0) return 8 * rb + x < ng.fn ? 8 * rb + x : kNone;
        if (kind == 1) return 4 * rb + x < ng.uc ? ng.ucol(4 * rb + x) : kNone;
        return ng.fn + x < ng.nn ? ng.fn + x : kNone;
    };
    auto b_idx = [&](uint32_t y) -> uint32_t {
        if (t == kNone) return kNone;
        if (kind == 0) return 8 * cb + y < ng.cf ? ng.fcol(8 * cb + y) : kNone;
        if (kind == 1) return 16 * cb + y < ng.fn ? 16 * cb + y : kNone;
        return 16 * cb + y < ng.l2 ? ng.l2col(16 * cb + y) : kNone;
    };
    uint32_t ra[R], rc[C];
#pragma unroll
    for (uint32_t x = 0; x < R; ++x) {
        const uint32_t i = a_idx(x);
        ra[x] = (i != kNone ? nd.id[i] : zero_row) * H;
    }
#pragma unroll
    for (uint32_t y = 0; y < C; ++y) {
        const uint32_t j = b_idx(y);
        rc[y] = (j != kNone ? nd.id[j] : zero_row) * H;
    }
    float2 acc[32];
    gl_tile<R, C, kF>(base, H, ra, rc, mz, acc);
    float row[8];
    group_reduce64(acc, l8, row);
    if (t == kNone) return;
    // this lane's 8 pairs: accumulator row X = floats 8X .. 8X + 7
    const uint32_t X = reduced_row(l8);
    const uint32_t p = a_idx(kF ? X : X >> 1);  // short-side candidate
    if (p == kNone) return;
    const uint32_t y0 = kF ? 0u : 8u * (X & 1u);  // first long-side index
    uint64_t* const D = c.D + doff;
#pragma unroll
    for (uint32_t y = 0; y < 8; ++y) {
        const uint32_t q = b_idx(y0 + y);
        if (q == kNone) continue;
        // new x new pairs once (j > i); U1 pairs are all valid
        if (kind != 1 && q < ng.nn && q <= p) continue;
        gl_propose(c, nd, D, ng.nn, ng.m, p, q, row[y]);
    }
}

__device__ __forceinline__ void gl_load_node(const CandView& c, GlNode& nd, uint32_t u,
                                             uint32_t nn, uint32_t no, uint32_t lane) {
    const size_t base = size_t(u) * 2 * c.cap;
    for (uint32_t p = lane; p < nn + no; p += 32) {
        const uint32_t pos = p < nn ? p : c.cap + p - nn;
        nd.id[p] = c.ids[base + pos];
        nd.mx[p] = c.filter ? c.cmax[base + pos] : __int_as_float(0x7f800000);
        nd.cnt[p] = 0;
    }
}

__device__ __forceinline__ void gl_flush_node(const CandView& c, const GlNode& nd, uint64_t doff,
                                              uint32_t nn, uint32_t no, uint32_t lane) {
    const uint32_t m = nn + no;
    for (uint32_t r = lane; r < m; r += 32) c.D[doff + prow(r, nn, m)] = nd.cnt[r];
}

__global__ void __launch_bounds__(kGlThreads, KNNG_GL_MINBLOCKS) join_gl_kernel(CandView c, const float* dl,
                                                                uint32_t S, uint32_t n,
                                                                IterCounters* ctr,
                                                                float minus_zero) {
    __shared__ GlShared sh;
    if (ctr->overflow || ctr->halt) return;
    const float2 mz = make_float2(minus_zero, minus_zero);  // -0.0f, opaque to ptxas
    const uint32_t lane = lane_id(), w = threadIdx.x >> 5, g = lane >> 3, l8 = lane & 7u;
    const uint32_t n_active = ctr->active;
    const uint32_t H = S / 16, zero_row = n;
    const char* const base = reinterpret_cast<const char*>(dl) + 8 * l8;
    GlNode* const nodes = sh.node[w];
    for (;;) {
        uint32_t a0 = 0;
        if (lane == 0) a0 = atomicAdd(&ctr->work, 4u);
        a0 = __shfl_sync(0xffffffffu, a0, 0);
        if (a0 >= n_active) break;
        uint4 rec = make_uint4(0, 0, 0, 0);
        const bool have = lane < 4 && a0 + lane < n_active;
        if (have) rec = c.arec[a0 + lane];
        const uint32_t nn_l = rec.y & 0xffffu;
        const uint32_t small = __ballot_sync(0xffffffffu, have && nn_l <= 4);
        const uint32_t big = __ballot_sync(0xffffffffu, have && nn_l > 4);
        // nodes with nn <= 4 (leftover rows only): one per group
        if (small) {
            const uint32_t ns = __popc(small);
            for (uint32_t s = 0; s < ns; ++s) {
                const uint32_t src = __fns(small, 0, s + 1);
                const uint32_t u = __shfl_sync(0xffffffffu, rec.x, src);
                const uint32_t y = __shfl_sync(0xffffffffu, rec.y, src);
                gl_load_node(c, nodes[s], u, y & 0xffffu, y >> 16, lane);
            }
            __syncwarp();
            const uint32_t src = g < ns ? __fns(small, 0, g + 1) : 0u;
            const uint32_t y = __shfl_sync(0xffffffffu, rec.y, src);
            const uint64_t doff = uint64_t(__shfl_sync(0xffffffffu, rec.z, src)) |
                                  (uint64_t(__shfl_sync(0xffffffffu, rec.w, src)) << 32);
            GlGeom ng;
            ng.set(g < ns ? y & 0xffffu : 0u, g < ns ? y >> 16 : 0u);
            uint32_t rounds = ng.nU2;
#pragma unroll
            for (uint32_t o = 8; o < 32; o <<= 1) rounds = max(rounds, __shfl_xor_sync(0xffffffffu, rounds, o));
            for (uint32_t r = 0; r < rounds; ++r)
                gl_run_tile<false>(c, nodes[g < ns ? g : 0], ng, doff, r < ng.nU2 ? r : kNone, base,
                                   zero_row, H, l8, mz);
            __syncwarp();
            for (uint32_t s = 0; s < ns; ++s) {
                const uint32_t src2 = __fns(small, 0, s + 1);
                const uint32_t y2 = __shfl_sync(0xffffffffu, rec.y, src2);
                const uint64_t off2 = uint64_t(__shfl_sync(0xffffffffu, rec.z, src2)) |
                                      (uint64_t(__shfl_sync(0xffffffffu, rec.w, src2)) << 32);
                gl_flush_node(c, nodes[s], off2, y2 & 0xffffu, y2 >> 16, lane);
            }
            __syncwarp();
        }
        // larger nodes: the whole warp, four tiles at a time
        for (uint32_t bits = big; bits; bits &= bits - 1u) {
            const uint32_t src = __ffs(bits) - 1u;
            const uint32_t u = __shfl_sync(0xffffffffu, rec.x, src);
            const uint32_t y = __shfl_sync(0xffffffffu, rec.y, src);
            const uint64_t doff = uint64_t(__shfl_sync(0xffffffffu, rec.z, src)) |
                                  (uint64_t(__shfl_sync(0xffffffffu, rec.w, src)) << 32);
            const uint32_t nn = y & 0xffffu, no = y >> 16;
            gl_load_node(c, nodes[0], u, nn, no, lane);
            __syncwarp();
            GlGeom ng;
            ng.set(nn, no);
            for (uint32_t t0 = 0; t0 < ng.nF; t0 += 4)
                gl_run_tile<true>(c, nodes[0], ng, doff, t0 + g < ng.nF ? t0 + g : kNone, base,
                                  zero_row, H, l8, mz);
            const uint32_t nU = ng.nU1 + ng.nU2;
            for (uint32_t t0 = 0; t0 < nU; t0 += 4)
                gl_run_tile<false>(c, nodes[0], ng, doff, t0 + g < nU ? t0 + g : kNone, base,
                                   zero_row, H, l8, mz);
            __syncwarp();
            gl_flush_node(c, nodes[0], doff, nn, no, lane);
            __syncwarp();
        }
    }
}

// Lane-major copy: row r, half-slab h, position 2 l + c <- element 16 h + 8 c + l
// (zero past the row stride); row n is all zero.  One thread per output float2.
__global__ void gl_pack_kernel(const float* __restrict__ data, uint32_t n, uint32_t stride,
                               uint32_t S, float2* __restrict__ dl) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;  // float2 index
    const size_t total = size_t(n + 1) * (S / 2);
    if (i >= total) return;
    const uint32_t r = uint32_t(i / (S / 2)), w = uint32_t(i % (S / 2));
    if (r == n) {  // the all-zero row that padding slots read
        dl[i] = make_float2(0.0f, 0.0f);
        return;
    }
    const uint32_t h = w / 8, l = w % 8;
    const uint32_t e0 = 16 * h + l, e1 = 16 * h + 8 + l;
    const float* row = data + size_t(r) * stride;
    dl[i] = make_float2(e0 < stride ? row[e0] : 0.0f, e1 < stride ? row[e1] : 0.0f);
}

}  // namespace

uint32_t gl_row_floats(uint32_t stride) { return (stride + 15u) / 16u * 16u; }

void launch_gl_pack(const float* data, uint32_t n, uint32_t stride, float* dl, cudaStream_t s) {
    const uint32_t S = gl_row_floats(stride);
    const size_t total = size_t(n + 1) * (S / 2);
    gl_pack_kernel<<<uint32_t((total + 255) / 256), 256, 0, s>>>(data, n, stride, S,
                                                                 reinterpret_cast<float2*>(dl));
}

void launch_join_gl(const CandView& c, const float* dl, uint32_t n, uint32_t stride,
                    IterCounters* ctr, uint32_t max_active, cudaStream_t s) {
    if (!max_active) return;
    static int per_sm[kMaxDevices] = {};
    int& occ = per_sm[current_device()];
    if (!occ) {
        int v = 0;
        check_launch(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, join_gl_kernel,
                                                                   int(kGlThreads), 0));
        occ = v < 1 ? 1 : v;
    }
    uint32_t grid = device_sm_count() * uint32_t(occ);
    const uint32_t need = (max_active + 4 * kGlWarps - 1) / (4 * kGlWarps);
    if (grid > need) grid = need;
    check_launch(cudaMemsetAsync(&ctr->work, 0, sizeof(uint32_t), s));
    join_gl_kernel<<<grid, kGlThreads, 0, s>>>(c, dl, gl_row_floats(stride), n, ctr, -0.0f);
}

}  // namespace knng_cuda
