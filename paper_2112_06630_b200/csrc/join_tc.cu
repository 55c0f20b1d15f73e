// Tensor-core-screened local join (compute_step, reference descent.hpp:82-153)
// for high-dimensional data after the first iteration.
//
// After iteration 1 most of a node's pairs cannot change the graph: a pair
// (a, b) matters only if its distance beats the iteration-start row maximum
// of a or of b (the join's prefilter, join.cu).  On C2/C5-like data ~90% of
// the pairs of iterations >= 2 fail that test (scripts/survivor_stats.py), yet
// the FP32 tile kernel evaluates every one of them exactly.  This kernel
//
//   1. bulk-loads (TMA 1-D copies) the node's whole candidate rows once into
//      a shared-memory arena and forms every new x candidate dot product on
//      the tensor cores (mma.sync m16n8k8 TF32, FP32 accumulate);
//   2. turns each into a rigorous LOWER bound of the reference's distance,
//      ||a||^2 + ||b||^2 - 2 (a.b + E) - slack with E = 2^-8 ||a|| ||b|| (TF32
//      truncation of both factors costs < 2^-9 ||a|| ||b||, FP32 accumulation
//      far less; 2x margin), scaled by (1 - 4 gamma) for the reference's own
//      FP32 rounding of sum (a_j - b_j)^2; a pair whose bound is >=
//      max(row maximum of a, of b) cannot be kept by the prefilter and is
//      dropped;
//   3. evaluates the surviving pairs EXACTLY as the reference does — 8 strided
//      lanes, FMA-contracted inside full 5x5 / triangular tiles and unfused
//      elsewhere (distance.hpp:29-190), the same lane tree — from the resident
//      rows, and writes the proposals that beat an endpoint's row maximum into
//      the node's proposal block in join.cu's format.
//
// The dropped pairs are exactly pairs the FP32 kernel's prefilter drops, so
// the proposal blocks carry the same keys and the merge gives the same rows
// (tests/test_gpu_screened.py).
//
// Warp roles (one CTA per SM, 288 threads): warp 8 is the producer — it
// claims active nodes, stages their slot tables (ids, row maxima, norms) and
// issues one bulk copy per candidate row into the arena, nodes queued ahead in
// kASlots slots (mbarriers full / empty per slot); warps 0-3 and 4-7 are two
// consumer groups taking alternate slots.  A node whose rows do not fit the
// arena goes to an overflow list that the FP32 kernel handles afterwards.
// Compiled with --fmad=false; exact arithmetic uses explicit intrinsics.
#include <cstdio>

#include "kernels.cuh"

namespace knng_cuda {

namespace {

#ifndef KNNG_TC_PROF
#define KNNG_TC_PROF 0  // 1: per-role clock totals (diagnostics build)
#endif
#if KNNG_TC_PROF
__device__ unsigned long long g_tc_prof[16];
#define TC_T0() long long tc_t = clock64()
#define TC_MARK(i)                                                         \
    do {                                                                   \
        const long long tn_ = clock64();                                   \
        if ((threadIdx.x & 127u) == 0 || threadIdx.x == 256)               \
            atomicAdd(&g_tc_prof[i], (unsigned long long)(tn_ - tc_t));    \
        tc_t = tn_;                                                        \
    } while (0)
#else
#define TC_T0() ((void)0)
#define TC_MARK(i) ((void)0)
#endif

constexpr uint32_t kAGroups = 2;                     // consumer groups of 4 warps
constexpr uint32_t kAGroupThreads = 128;
constexpr uint32_t kAThreads = kAGroups * kAGroupThreads + 32;  // + producer warp
constexpr uint32_t kASlots = 4;                      // nodes in flight (2 per group)
constexpr uint32_t kAMaxM = 2 * kMaxCap;             // candidates of one node
constexpr uint32_t kARound = kAGroupThreads;         // survivor pairs per exact round
constexpr uint32_t kASurvWords = kAMaxM / 32;        // bitmask words per new row
constexpr uint32_t kASentinel = 0xffffffffu;

struct SlotTab {
    uint32_t rid[kAMaxM];  // combined index -> data row
    float rmx[kAMaxM];     // row maximum of the candidate (iteration start)
    float rn2[kAMaxM];     // ||x||^2 rounded down
    float rnu[kAMaxM];     // ||x|| rounded up
    uint4 rec;             // {u, nn | no << 16, doff lo, doff hi}; rec.y = sentinel: stop
    uint32_t off;          // arena float offset of row 0
    uint32_t pad[3];
};

struct GroupTab {
    // survivor bitmasks, row i = new candidate i: fused-path pairs (first
    // nn * kASurvWords words), then unfused, so the rounds take them in order
    uint32_t surv[2 * kMaxCap * kASurvWords];
    uint32_t rowcnt[kAMaxM];
    uint16_t plist[kARound];
    uint32_t nsurv, npairs, nfused, cursor;
};

struct ArenaShared {
    uint64_t full[kASlots], empty[kASlots];
    SlotTab slot[kASlots];
    GroupTab grp[kAGroups];
};

constexpr size_t kAArenaOffset = (sizeof(ArenaShared) + 127) / 128 * 128;
constexpr size_t kASmemMax = 227 * 1024;  // sm_100 opt-in maximum per block

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// Waits for the phase with the given parity; the suspend-time hint lets the
// hardware park the waiting warp instead of spinning on issue slots the
// computing warps need.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n TC_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        " @!p bra TC_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
// One 1-D bulk copy (TMA engine): `bytes` (multiple of 16) from global to
// shared memory, completing on the mbarrier as transaction bytes.
__device__ __forceinline__ void bulk_g2s(float* dst, const float* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void group_sync(uint32_t grp) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "r"(kAGroupThreads) : "memory");
}

__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ size_t tc_prow(uint32_t r, uint32_t nn, uint32_t m) {
    return r < nn ? size_t(r) * m : size_t(nn) * m + size_t(r - nn) * (nn + 1);
}

// Rows staged for a node: enough for the m16 x n8 tiles (pads are read, never
// used).  The arena row pitch is stride + 4 floats: 8 rows x 4 columns of an
// MMA fragment then fall in 32 distinct banks (stride % 8 == 0).
__host__ __device__ __forceinline__ uint32_t staged_rows(uint32_t nn, uint32_t m) {
    const uint32_t a = 16 * ((nn + 15) / 16), b = 8 * ((m + 7) / 8);
    return a > b ? a : b;
}

// Screening for a node with NMI 16-row blocks of new candidates: warp w of the
// group owns column blocks nj = w + 4 q (q < 4) of every row block over the
// whole row; each thread then holds its C elements (rows 16 mi + g (+8),
// columns 8 nj + 2 t (+1)) and sets the survivor bits of its pairs.
template <uint32_t NMI>
__device__ __forceinline__ uint32_t screen_node(const float* rows, uint32_t pitch,
                                                uint32_t stride, const SlotTab& T, GroupTab& G,
                                                uint32_t nn, uint32_t no, float lb_scale) {
    // KK independent accumulator chains per tile along K (k-step ks feeds
    // chain ks % KK): the legacy MMA's latency is long on sm_100
    constexpr uint32_t KK = NMI == 1 ? 4 : NMI == 2 ? 2 : 1;
    const uint32_t gtid = threadIdx.x % kAGroupThreads, warp = gtid >> 5, lane = gtid & 31u;
    const uint32_t g = lane >> 2, t = lane & 3u, m = nn + no, nnj = (m + 7) / 8;
    const uint32_t nq = nnj > warp ? (nnj - warp + 3) / 4 : 0;
    float acc[4][NMI][4];
    float part[KK > 1 ? KK - 1 : 1][4][NMI][4];
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q)
#pragma unroll
        for (uint32_t mi = 0; mi < NMI; ++mi)
#pragma unroll
            for (uint32_t r = 0; r < 4; ++r) {
                acc[q][mi][r] = 0.0f;
#pragma unroll
                for (uint32_t kk = 0; kk + 1 < KK; ++kk) part[kk][q][mi][r] = 0.0f;
            }
    auto kstep = [&](uint32_t k0, float (&A)[4][NMI][4]) {
        uint32_t a[NMI][4];
        const float* pa0 = rows + g * pitch + t + k0;
#pragma unroll
        for (uint32_t mi = 0; mi < NMI; ++mi) {
            const float* pa = pa0 + 16 * mi * pitch;
            a[mi][0] = __float_as_uint(pa[0]);
            a[mi][1] = __float_as_uint(pa[8 * pitch]);
            a[mi][2] = __float_as_uint(pa[4]);
            a[mi][3] = __float_as_uint(pa[8 * pitch + 4]);
        }
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
            if (q < nq) {
                const float* pb = pa0 + 8 * (warp + 4 * q) * pitch;
                const uint32_t b0 = __float_as_uint(pb[0]), b1 = __float_as_uint(pb[4]);
#pragma unroll
                for (uint32_t mi = 0; mi < NMI; ++mi) mma_tf32(A[q][mi], a[mi], b0, b1);
            }
        }
    };
    if (nq > 0) {
        uint32_t k0 = 0;
        for (; k0 + 8 * KK <= stride; k0 += 8 * KK) {
            kstep(k0, acc);
#pragma unroll
            for (uint32_t kk = 0; kk + 1 < KK; ++kk) kstep(k0 + 8 * (kk + 1), part[kk]);
        }
        for (; k0 < stride; k0 += 8) kstep(k0, acc);
#pragma unroll
        for (uint32_t kk = 0; kk + 1 < KK; ++kk)
#pragma unroll
            for (uint32_t q = 0; q < 4; ++q)
#pragma unroll
                for (uint32_t mi = 0; mi < NMI; ++mi)
#pragma unroll
                    for (uint32_t r = 0; r < 4; ++r) acc[q][mi][r] += part[kk][q][mi][r];
    }
    // lower bounds -> survivor bits.  Path of a pair (distance.hpp /
    // descent.hpp:107-147): new x new (i < j) inside the triangle tiles iff
    // j < fn; new x old inside a full 5x5 block iff i < fn and j - nn < fo
    const uint32_t fn = nn - nn % 5, fo = no - no % 5, nwords = nn * kASurvWords;
    uint32_t mine = 0;
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) {
        if (q >= nq) continue;
#pragma unroll
        for (uint32_t mi = 0; mi < NMI; ++mi)
#pragma unroll
            for (uint32_t r = 0; r < 4; ++r) {
                const uint32_t i = 16 * mi + g + 8 * (r >> 1);
                const uint32_t j = 8 * (warp + 4 * q) + 2 * t + (r & 1u);
                if (i >= nn || j >= m || (j < nn && j <= i)) continue;
                if (T.rid[i] == T.rid[j]) continue;  // self pair: try_insert ignores it
                const float dot = acc[q][mi][r];
                const float s2 = T.rn2[i] + T.rn2[j];
                const float e = 0.00390625f * T.rnu[i] * T.rnu[j];  // 2^-8 ||a|| ||b||
                const float slack = 9.5367431640625e-07f * (s2 + 2.0f * fabsf(dot) + 2.0f * e);
                const float lb = (s2 - 2.0f * dot - 2.0f * e - slack) * lb_scale;
                if (!(lb >= fmaxf(T.rmx[i], T.rmx[j]))) {
                    const bool f = j < nn ? j < fn : (i < fn && j - nn < fo);
                    atomicOr(&G.surv[(f ? 0u : nwords) + i * kASurvWords + (j >> 5)],
                             1u << (j & 31u));
                    ++mine;
                }
            }
    }
    return mine;
}

// Warp 0 of a group: the next <= kARound surviving pairs (fused ones first),
// cleared from the bitmasks, into G.plist; G.npairs / G.nfused / G.cursor.
__device__ __forceinline__ void pick_round(GroupTab& G, uint32_t nwords) {
    const uint32_t lane = threadIdx.x & 31u, total_words = 2 * nwords;
    uint32_t np = 0, nf = 0, base = G.cursor;
    for (; base < total_words && np < kARound; base += 32) {
        const uint32_t w = base + lane;
        uint32_t bits = w < total_words ? G.surv[w] : 0u;
        const uint32_t cnt = __popc(bits);
        uint32_t incl = cnt;
#pragma unroll
        for (uint32_t o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const uint32_t excl = incl - cnt, room = kARound - np;
        const uint32_t take = excl < room ? min(cnt, room - excl) : 0u;
        const uint32_t wl = w < nwords ? w : w - nwords;
        const uint32_t i = wl / kASurvWords, jb = (wl % kASurvWords) * 32;
        uint32_t slot = np + excl;
        for (uint32_t q = 0; q < take; ++q) {
            const uint32_t b = __ffs(bits) - 1;
            bits &= bits - 1;
            G.plist[slot++] = uint16_t((i << 7) | (jb + b));
        }
        if (w < total_words) G.surv[w] = bits;
        uint32_t f = w < nwords ? take : 0u;
#pragma unroll
        for (uint32_t o = 16; o > 0; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
        nf += f;
        np += min(__shfl_sync(0xffffffffu, incl, 31), room);
    }
    __syncwarp();
    // resume at the first non-empty word
    uint32_t cur = G.cursor;
    for (;;) {
        const uint32_t w = cur + lane;
        const uint32_t b = __ballot_sync(0xffffffffu, w < total_words && G.surv[w] != 0u);
        if (b) {
            cur += __ffs(b) - 1;
            break;
        }
        cur += 32;
        if (cur >= total_words) {
            cur = total_words;
            break;
        }
    }
    if (lane == 0) {
        G.npairs = np;
        G.nfused = nf;
        G.cursor = cur;
    }
}

// Exact distance of one pair (rows pa, pb resident), all 8 reference lanes in
// registers: lane l = elements 8c + l, packed FP32x2 on lane pairs.
template <bool kFused>
__device__ __forceinline__ float exact_pair(const float* pa, const float* pb, uint32_t stride,
                                            float2 mz2) {
    const float2 m1 = make_float2(-1.0f, -1.0f);
    float2 acc[4];
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) acc[q] = make_float2(0.0f, 0.0f);
#pragma unroll 4
    for (uint32_t c = 0; c < stride / 8; ++c) {
        const float4 a0 = *reinterpret_cast<const float4*>(pa + 8 * c);
        const float4 a1 = *reinterpret_cast<const float4*>(pa + 8 * c + 4);
        const float4 b0 = *reinterpret_cast<const float4*>(pb + 8 * c);
        const float4 b1 = *reinterpret_cast<const float4*>(pb + 8 * c + 4);
        float2 d[4];  // a - b exactly: fma(b, -1, a)
        d[0] = __ffma2_rn(make_float2(b0.x, b0.y), m1, make_float2(a0.x, a0.y));
        d[1] = __ffma2_rn(make_float2(b0.z, b0.w), m1, make_float2(a0.z, a0.w));
        d[2] = __ffma2_rn(make_float2(b1.x, b1.y), m1, make_float2(a1.x, a1.y));
        d[3] = __ffma2_rn(make_float2(b1.z, b1.w), m1, make_float2(a1.z, a1.w));
        if (kFused) {
#pragma unroll
            for (uint32_t q = 0; q < 4; ++q) acc[q] = __ffma2_rn(d[q], d[q], acc[q]);
        } else {
            // the rounded square as fma(d, d, -0) with an opaque -0 (join.cu
            // tile_slab), then a packed add
#pragma unroll
            for (uint32_t q = 0; q < 4; ++q) acc[q] = __fadd2_rn(acc[q], __ffma2_rn(d[q], d[q], mz2));
        }
    }
    // the reference's lane tree ((0+1)+(2+3))+((4+5)+(6+7))
    return __fadd_rn(__fadd_rn(__fadd_rn(acc[0].x, acc[0].y), __fadd_rn(acc[1].x, acc[1].y)),
                     __fadd_rn(__fadd_rn(acc[2].x, acc[2].y), __fadd_rn(acc[3].x, acc[3].y)));
}

__global__ void __launch_bounds__(kAThreads, 1) join_tc_kernel(GraphView g, CandView c,
                                                               IterCounters* ctr,
                                                               const float* __restrict__ nrm2,
                                                               const float* __restrict__ nrmu,
                                                               uint4* ovf, IterCounters* octr,
                                                               uint32_t arena_floats,
                                                               float lb_scale, float minus_zero) {
    extern __shared__ __align__(128) unsigned char tc_smem[];
    ArenaShared& sh = *reinterpret_cast<ArenaShared*>(tc_smem);
    float* const arena = reinterpret_cast<float*>(tc_smem + kAArenaOffset);
    const uint32_t tid = threadIdx.x, stride = g.stride, pitch = stride + 4, cap = c.cap;
    if (tid == 0) {
        for (uint32_t s = 0; s < kASlots; ++s) {
            mbar_init(&sh.full[s], 1);
            mbar_init(&sh.empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (ctr->overflow || ctr->halt) return;  // the proposal blocks outgrew their buffer
    const uint32_t n_active = ctr->active;

    if (tid >= kAGroups * kAGroupThreads) {
        // ---------------- producer warp ----------------
        const uint32_t lane = tid & 31u;
        uint32_t head = 0;                            // next free arena float
        uint32_t reg_off[kASlots], reg_len[kASlots];  // arena regions of in-use slots
        uint32_t in_use = 0, epar = 0;                // slot bits; empty-barrier parities
#pragma unroll
        for (uint32_t s = 0; s < kASlots; ++s) reg_off[s] = reg_len[s] = 0;
        auto release = [&](uint32_t s) {  // wait for slot s's consumer group
            mbar_wait(&sh.empty[s], (epar >> s) & 1u);
            epar ^= 1u << s;
            in_use &= ~(1u << s);
        };
        uint32_t k = 0, ended = 0;
        TC_T0();
        while (ended < kAGroups) {
            uint32_t a = 0;
            if (lane == 0) a = atomicAdd(&ctr->work, 1u);
            a = __shfl_sync(0xffffffffu, a, 0);
            uint4 rec = make_uint4(0, kASentinel, 0, 0);
            uint32_t nn = 0, m = 0, len = 0;
            if (a < n_active) {
                rec = c.arec[a];
                nn = rec.y & 0xffffu;
                m = nn + (rec.y >> 16);
                TC_MARK(0);
                len = staged_rows(nn, m) * pitch;
                if (len > arena_floats) {  // too large for the arena: FP32 kernel
                    if (lane == 0) ovf[atomicAdd(&octr->active, 1u)] = rec;
                    continue;
                }
            }
            // slot k must be free, and so must every slot whose region meets
            // [off, off + len) (regions are allocated in slot order)
            if ((in_use >> k) & 1u) release(k);
            uint32_t off = 0;
            if (len) {
                off = head + len <= arena_floats ? head : 0u;
#pragma unroll
                for (uint32_t s = 0; s < kASlots; ++s)
                    if (((in_use >> s) & 1u) && reg_off[s] < off + len &&
                        off < reg_off[s] + reg_len[s])
                        release(s);
                head = off + len;
            }
            TC_MARK(1);
            SlotTab& T = sh.slot[k];
            for (uint32_t x = lane; x < m; x += 32) {
                const size_t pos = size_t(rec.x) * 2 * cap + (x < nn ? x : cap + x - nn);
                const uint32_t id = c.ids[pos];
                T.rid[x] = id;
                T.rmx[x] = c.cmax[pos];
                T.rn2[x] = nrm2[id];
                T.rnu[x] = nrmu[id];
            }
            if (lane == 0) {
                T.rec = rec;
                T.off = off;
            }
            __syncwarp();
            TC_MARK(2);
            if (len) {
                // the arena region was last used through the generic proxy
                fence_proxy_async();
                if (lane == 0) mbar_expect_tx(&sh.full[k], m * stride * 4u);
                __syncwarp();
                for (uint32_t x = lane; x < m; x += 32)
                    bulk_g2s(arena + off + x * pitch, g.data + size_t(T.rid[x]) * stride,
                             stride * 4u, &sh.full[k]);
            } else {
                if (lane == 0) mbar_arrive(&sh.full[k]);  // stop marker for its group
                ++ended;
            }
            TC_MARK(3);
            in_use |= 1u << k;
            reg_off[k] = off;
            reg_len[k] = len;
            k = k + 1 == kASlots ? 0 : k + 1;
        }
        return;
    }

    // ---------------- consumer groups ----------------
    const uint32_t grp = tid / kAGroupThreads, gtid = tid % kAGroupThreads;
    GroupTab& G = sh.grp[grp];
    const float2 mz2 = make_float2(minus_zero, minus_zero);  // -0.0f, opaque to ptxas
    unsigned long long st_pairs = 0, st_surv = 0;
    uint32_t fpar = 0;
    TC_T0();
    for (uint32_t k = grp;; k = (k + kAGroups) % kASlots) {
        mbar_wait(&sh.full[k], (fpar >> k) & 1u);
        fpar ^= 1u << k;
        TC_MARK(4);
        const SlotTab& T = sh.slot[k];
        const uint4 rec = T.rec;
        if (rec.y == kASentinel) break;
        const uint32_t nn = rec.y & 0xffffu, no = rec.y >> 16, m = nn + no;
        const unsigned long long doff = uint64_t(rec.z) | (uint64_t(rec.w) << 32);
        const float* const rows = arena + T.off;
        const uint32_t nwords = nn * kASurvWords;
        for (uint32_t w = gtid; w < 2 * nwords; w += kAGroupThreads) G.surv[w] = 0;
        if (gtid < m) G.rowcnt[gtid] = 0;
        if (gtid == 0) {
            G.nsurv = 0;
            G.cursor = 0;
        }
        group_sync(grp);
        // ---- 1-2. screening dot products on the tensor cores, lower bounds ----
        uint32_t mine = 0;
        switch ((nn + 15) / 16) {
            case 1: mine = screen_node<1>(rows, pitch, stride, T, G, nn, no, lb_scale); break;
            case 2: mine = screen_node<2>(rows, pitch, stride, T, G, nn, no, lb_scale); break;
            case 3: mine = screen_node<3>(rows, pitch, stride, T, G, nn, no, lb_scale); break;
            default: mine = screen_node<4>(rows, pitch, stride, T, G, nn, no, lb_scale); break;
        }
#pragma unroll
        for (uint32_t o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
        if ((gtid & 31u) == 0 && mine) atomicAdd(&G.nsurv, mine);
        group_sync(grp);
        TC_MARK(5);
        // ---- 3. exact evaluation of the survivors, one pair per thread ----
        uint32_t left = G.nsurv;
        if (gtid == 0) {
            st_pairs += nn * (nn - 1) / 2 + nn * no;
            st_surv += left;
        }
        uint64_t* const D = c.D + doff;
        while (left > 0) {
            if (gtid < 32) pick_round(G, nwords);
            group_sync(grp);
            const uint32_t np = G.npairs;
            if (gtid < np) {
                const uint32_t code = G.plist[gtid];
                const uint32_t i = code >> 7, j = code & 127u;
                const float dist =
                    gtid < G.nfused
                        ? exact_pair<true>(rows + i * pitch, rows + j * pitch, stride, mz2)
                        : exact_pair<false>(rows + i * pitch, rows + j * pitch, stride, mz2);
                if (dist < T.rmx[i]) {
                    const uint32_t pos = atomicAdd(&G.rowcnt[i], 1u);
                    D[tc_prow(i, nn, m) + 1 + pos] = pack_key(dist, T.rid[j]);
                }
                if (dist < T.rmx[j]) {
                    const uint32_t pos = atomicAdd(&G.rowcnt[j], 1u);
                    D[tc_prow(j, nn, m) + 1 + pos] = pack_key(dist, T.rid[i]);
                }
            }
            left = np < left && np > 0 ? left - np : 0u;
            group_sync(grp);  // plist reused; row counters settled
        }
        TC_MARK(6);
        // row counts of the node's proposal block; the slot goes back
        if (gtid < m) D[tc_prow(gtid, nn, m)] = G.rowcnt[gtid];
        group_sync(grp);
        if (gtid == 0) mbar_arrive(&sh.empty[k]);
        TC_MARK(7);
    }
    if (gtid == 0 && st_pairs) {
        atomicAdd(&ctr->screened, st_pairs);
        atomicAdd(&ctr->survivors, st_surv);
    }
}

// ||x||^2 rounded down and ||x|| rounded up per row (double accumulation):
// the screening bound's inputs.  One warp per row.
__global__ void row_norms_kernel(const float* __restrict__ data, uint32_t n, uint32_t stride,
                                 float* nrm2, float* nrmu) {
    const uint32_t row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31u;
    if (row >= n) return;
    const float4* p = reinterpret_cast<const float4*>(data + size_t(row) * stride);
    double s = 0.0;
    for (uint32_t q = lane; q < stride / 4; q += 32) {
        const float4 v = p[q];
        s += double(v.x) * v.x + double(v.y) * v.y + double(v.z) * v.z + double(v.w) * v.w;
    }
#pragma unroll
    for (uint32_t o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        nrm2[row] = __double2float_rd(s);
        nrmu[row] = __double2float_ru(sqrt(s) * (1.0 + 1e-15));
    }
}

}  // namespace

void launch_row_norms(const float* data, uint32_t n, uint32_t stride, float* nrm2, float* nrmu,
                      cudaStream_t s) {
    row_norms_kernel<<<uint32_t((size_t(n) * 32 + 255) / 256), 256, 0, s>>>(data, n, stride, nrm2,
                                                                            nrmu);
}

void launch_join_tc(const GraphView& g, const CandView& c, IterCounters* ctr, uint32_t max_active,
                    const float* nrm2, const float* nrmu, uint4* ovf, IterCounters* octr,
                    cudaStream_t s) {
    if (!max_active) return;
    static bool attrs[kMaxDevices] = {};
    bool& attr = attrs[current_device()];
    if (!attr) {
        check_launch(cudaFuncSetAttribute(join_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(kASmemMax)));
        attr = true;
    }
    const uint32_t arena_floats = uint32_t((kASmemMax - kAArenaOffset) / sizeof(float));
    // the reference's FP32 sum of (a_j - b_j)^2 over 8 lanes of stride / 8
    // terms plus the 3-level tree is within (stride / 8 + 3) 2^-24 of the real
    // value (non-negative terms); the bound is scaled by 1 - 4x that
    const double gamma = (double(g.stride) / 8.0 + 3.0) * 5.9604644775390625e-08;
    const float lb_scale = float(1.0 - 4.0 * gamma);
    check_launch(cudaMemsetAsync(&ctr->work, 0, sizeof(uint32_t), s));
    check_launch(cudaMemsetAsync(octr, 0, sizeof(IterCounters), s));
    uint32_t grid = device_sm_count();
    if (grid > max_active) grid = max_active;
    join_tc_kernel<<<grid, kAThreads, kASmemMax, s>>>(g, c, ctr, nrm2, nrmu, ovf, octr,
                                                      arena_floats, lb_scale, -0.0f);
    // nodes too large for the arena: the FP32 tile kernel over the overflow list
    CandView co = c;
    co.arec = ovf;
    launch_join_distances(g, co, nullptr, octr, max_active, s);
#if KNNG_TC_PROF
    unsigned long long h[16];
    cudaMemcpyFromSymbolAsync(h, g_tc_prof, sizeof(h), 0, cudaMemcpyDeviceToHost, s);
    IterCounters ho;
    check_launch(cudaMemcpyAsync(&ho, octr, sizeof(ho), cudaMemcpyDeviceToHost, s));
    cudaStreamSynchronize(s);
    const double G = grid;
    fprintf(stderr,
            "[tc prof] per CTA kcyc: producer claim %.0f release %.0f tables %.0f issue %.0f | "
            "consumers(2) wait %.0f screen %.0f exact %.0f tail %.0f | overflow nodes %u\n",
            h[0] / G / 1e3, h[1] / G / 1e3, h[2] / G / 1e3, h[3] / G / 1e3, h[4] / G / 1e3,
            h[5] / G / 1e3, h[6] / G / 1e3, h[7] / G / 1e3, ho.active);
    const unsigned long long z[16] = {};
    cudaMemcpyToSymbolAsync(g_tc_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, s);
#endif
}

}  // namespace knng_cuda
