// Byte-valued local join on the 5th-generation tensor cores: TMA gather ->
// shared memory -> tcgen05.mma kind::i8 -> TMEM -> tcgen05.ld epilogue.
//
// Same contract and arithmetic as join_u8_kernel (join_u8.cu): every
// coordinate is an integer in [0, 255], so each of the reference's eight
// strided lane sums (distance.hpp:35-88) is the exact integer
//     lane_l(a, b) = |a|_l^2 + |b|_l^2 - 2 <a, b>_l
// and the reference's distance is the FP32 tree ((0+1)+(2+3))+((4+5)+(6+7)) of
// those lane sums — bit-identical to compute_step (descent.hpp:82-153).  Here
// the eight per-lane dot-product matrices of a node come from tcgen05 with
// their operands in shared memory instead of register fragments reloaded from
// L2 (the IMMA kernel is bound by those reloads: L1/TEX 98%,
// profiles/round1_ncu_join_u8_c2_iter1.json).
//
// One CTA (128 threads) per SM, one active node at a time, two node buffers:
//  * staging: thread 0 issues TMA gather4 copies (cp.async.bulk.tensor
//    .tile::gather4: four rows by index per instruction) of the node's m
//    candidate rows, lane segment by lane segment, from the lane-major byte
//    copy (8 x Kl bytes per row, Kl = 128) into a 128B-swizzled K-major tile
//    per lane (rows at 128-byte pitch) — the canonical SWIZZLE_128B UMMA
//    operand layout; the next node's rows load while this node computes;
//  * MMA: thread 0 issues, per column chunk q of 32 new candidates and per
//    reference lane l, Kl / 32 tcgen05.mma.cta_group::1.kind::i8 (M = 128
//    candidate rows, N = 32 new candidates, K = 32 bytes), D_l in TMEM
//    columns [32 l, 32 l + 32); tcgen05.commit signals an mbarrier;
//  * epilogue: thread i owns candidate row i (TMEM lane i): eight
//    tcgen05.ld 32x32b.x32 per chunk, the lane sums and the tree, and the
//    proposals that beat an endpoint's row maximum, written into the node's
//    proposal block in join.cu's format.
// A lane's A operand is 128 rows from its tile start; rows past the node's m
// read the next lane's tile (results ignored), the last lane has a full
// 128-row window.  Taken for Kl = 128 (stride <= 1024, e.g. C2) and
// max_candidates <= 52; otherwise the IMMA kernel runs.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>

#include "kernels.cuh"

namespace knng_cuda {

namespace {

#ifndef KNNG_U8TC_PROF
#define KNNG_U8TC_PROF 0  // 1: per-phase clock totals of thread 0 (diagnostics build)
#endif
#if KNNG_U8TC_PROF
__device__ unsigned long long g_u8tc_prof[8];
#define TP_T0() long long tp_t = clock64()
#define TP_MARK(i)                                                                    \
    do {                                                                              \
        const long long tn_ = clock64();                                              \
        if (threadIdx.x == 0) atomicAdd(&g_u8tc_prof[i], (unsigned long long)(tn_ - tp_t)); \
        tp_t = tn_;                                                                   \
    } while (0)
#else
#define TP_T0() ((void)0)
#define TP_MARK(i) ((void)0)
#endif
constexpr uint32_t kTThreads = 128;
constexpr uint32_t kTKl = 128;             // bytes per reference lane (one SW128 atom row)
constexpr uint32_t kTMaxRows = 104;        // ceil8(2 * 52)
#ifndef KNNG_U8TC_N
#define KNNG_U8TC_N 64
#endif
constexpr uint32_t kTChunk = KNNG_U8TC_N;  // new candidates per MMA column chunk (N)
constexpr uint32_t kTSub = 32;             // columns per epilogue pass
constexpr uint32_t kTTmemCols = 8 * kTChunk;  // eight lane accumulators
constexpr uint32_t kTLaneTile = kTMaxRows * kTKl;              // bytes per lane tile
constexpr uint32_t kTBuf = 7 * kTLaneTile + 128 * kTKl;        // last lane: 128-row window

struct TMeta {
    uint32_t id[kTMaxRows];
    float mx[kTMaxRows];
    int32_t nrm[kTMaxRows][8];
    uint4 rec;  // {u, nn | no << 16, doff lo, doff hi}; rec.y == ~0: none
};

struct TShared {
    uint64_t full[2];  // TMA completion per node buffer
    uint64_t mma;      // tcgen05.commit per column chunk
    uint32_t tmem;     // TMEM base address
    uint32_t next;     // next claimed active index
    uint32_t cnt[kTMaxRows];
    TMeta meta[2];
};

constexpr size_t kTMetaBytes = (sizeof(TShared) + 1023) / 1024 * 1024;
constexpr size_t kTSmem = kTMetaBytes + 2 * size_t(kTBuf) + 1024;  // + alignment slack
static_assert(kTSmem <= 232448, "tcgen05 byte join shared memory over the sm_100 limit");

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void t_mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void t_mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void t_mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n T_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra T_WAIT_%=;\n}\n" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
// four rows (byte rows r0..r3 of the lane-major copy) x 128 bytes from byte
// column col into dst (512 bytes, 128B swizzle by the destination address)
__device__ __forceinline__ void t_gather4(void* dst, const CUtensorMap* map, uint32_t col,
                                          uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3,
                                          uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
        "r"(su32(bar))
        : "memory");
}
// UMMA shared-memory descriptor, K-major, SWIZZLE_128B: 8-row groups 1024
// bytes apart (SBO), rows 128 bytes apart inside the atom, version 1 (sm_100)
__device__ __forceinline__ uint64_t t_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3fffu);         // start address
    d |= uint64_t(1u) << 16;                       // leading byte offset (unused, SW128 K-major)
    d |= uint64_t(1024u >> 4) << 32;               // stride byte offset
    d |= uint64_t(1u) << 46;                       // descriptor version
    d |= uint64_t(2u) << 61;                       // SWIZZLE_128B
    return d;
}
// instruction descriptor: kind::i8, A/B unsigned 8-bit K-major, D s32,
// M = 128, N = kTChunk
constexpr uint32_t kTIdesc = (2u << 4) | ((kTChunk >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void t_mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n"
        " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %4, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(accumulate), "r"(kTIdesc)
        : "memory");
}
__device__ __forceinline__ void t_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     su32(bar))
                 : "memory");
}
__device__ __forceinline__ void t_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void t_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// 32 consecutive TMEM columns of this thread's lane
__device__ __forceinline__ void t_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ size_t t_prow(uint32_t r, uint32_t nn, uint32_t m) {
    return r < nn ? size_t(r) * m : size_t(nn) * m + size_t(r - nn) * (nn + 1);
}

__global__ void __launch_bounds__(kTThreads, 1) join_u8_tc_kernel(
    const __grid_constant__ CUtensorMap map, CandView c, IterCounters* ctr,
    const int32_t* __restrict__ lnorm) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte aligned base for the swizzled tiles
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    TShared& sh = *reinterpret_cast<TShared*>(base);
    unsigned char* tiles = base + kTMetaBytes;
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    if (ctr->overflow || ctr->halt) return;
    const uint32_t n_active = ctr->active, cap = c.cap;

    if (tid == 0) {
        t_mbar_init(&sh.full[0], 1);
        t_mbar_init(&sh.full[1], 1);
        t_mbar_init(&sh.mma, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        sh.next = atomicAdd(&ctr->work, 1u);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         su32(&sh.tmem)),
                     "n"(kTTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    t_fence_before();
    __syncthreads();
    t_fence_after();
    const uint32_t tmem = sh.tmem;

    // node metadata into meta[b] (every thread), claimed index a
    auto load_meta = [&](uint32_t b, uint32_t a) {
        TMeta& M = sh.meta[b];
        if (a >= n_active) {
            if (tid == 0) M.rec = make_uint4(0, 0xffffffffu, 0, 0);
            return;
        }
        const uint4 rec = c.arec[a];
        const uint32_t u = rec.x, nn = rec.y & 0xffffu, m = nn + (rec.y >> 16);
        if (tid == 0) M.rec = rec;
        if (tid < kTMaxRows) {
            const uint32_t x = tid < m ? tid : 0u;  // padding rows: candidate 0 (read, unused)
            const size_t pos = size_t(u) * 2 * cap + (x < nn ? x : cap + x - nn);
            const uint32_t id = c.ids[pos];
            M.id[tid] = id;
            M.mx[tid] = c.filter ? c.cmax[pos] : __int_as_float(0x7f800000);
            const int4 n0 = __ldg(reinterpret_cast<const int4*>(lnorm + size_t(id) * 8));
            const int4 n1 = __ldg(reinterpret_cast<const int4*>(lnorm + size_t(id) * 8) + 1);
            M.nrm[tid][0] = n0.x;
            M.nrm[tid][1] = n0.y;
            M.nrm[tid][2] = n0.z;
            M.nrm[tid][3] = n0.w;
            M.nrm[tid][4] = n1.x;
            M.nrm[tid][5] = n1.y;
            M.nrm[tid][6] = n1.z;
            M.nrm[tid][7] = n1.w;
        }
    };
    // warp 0: the TMA gathers of meta[b]'s rows into tile buffer b, thread l
    // of the warp issuing reference lane l's (the expected byte count is
    // posted first, by thread 0)
    auto stage = [&](uint32_t b) {
        const TMeta& M = sh.meta[b];
        const uint32_t nn = M.rec.y & 0xffffu, m = nn + (M.rec.y >> 16);
        const uint32_t rows = (m + 7) / 8 * 8;
        unsigned char* buf = tiles + size_t(b) * kTBuf;
        if (tid == 0) t_mbar_expect(&sh.full[b], 8 * rows * kTKl);
        __syncwarp();
        if (tid < 8)
            for (uint32_t r = 0; r < rows; r += 4)
                t_gather4(buf + tid * kTLaneTile + r * kTKl, &map, tid * kTKl, M.id[r],
                          M.id[r + 1], M.id[r + 2], M.id[r + 3], &sh.full[b]);
    };

    load_meta(0, sh.next);
    __syncthreads();
    if (warp == 0 && sh.meta[0].rec.y != 0xffffffffu) stage(0);
    uint32_t k = 0, mma_phase = 0;
    TP_T0();
    for (;; ++k) {
        const uint32_t b = k & 1u;
        TMeta& M = sh.meta[b];
        if (M.rec.y == 0xffffffffu) break;
        // claim and stage the next node while this one computes
        if (tid == 0) sh.next = atomicAdd(&ctr->work, 1u);
        __syncthreads();
        load_meta(b ^ 1u, sh.next);
        if (tid < kTMaxRows) sh.cnt[tid] = 0;
        __syncthreads();
        TP_MARK(0);  // claim + next node's metadata
        if (warp == 0 && sh.meta[b ^ 1u].rec.y != 0xffffffffu) stage(b ^ 1u);
        TP_MARK(1);  // TMA issue
        const uint32_t nn = M.rec.y & 0xffffu, m = nn + (M.rec.y >> 16);
        uint64_t* const D = c.D + (uint64_t(M.rec.z) | (uint64_t(M.rec.w) << 32));
        t_mbar_wait(&sh.full[b], (k >> 1) & 1u);
        TP_MARK(2);  // waiting for this node's rows
        const uint32_t tile0 = su32(tiles + size_t(b) * kTBuf);
        // my candidate row, its id / bound / lane norms
        const uint32_t i = tid;
        const bool row_ok = i < m;
        const uint32_t id_i = row_ok ? M.id[i] : 0u;
        const float mx_i = row_ok ? M.mx[i] : 0.0f;
        int32_t na[8];
#pragma unroll
        for (uint32_t l = 0; l < 8; ++l) na[l] = row_ok ? M.nrm[i][l] : 0;
        for (uint32_t q = 0; q * kTChunk < nn; ++q) {
            if (tid == 0) {
                t_fence_after();
#pragma unroll
                for (uint32_t l = 0; l < 8; ++l) {
                    const uint32_t a_addr = tile0 + l * kTLaneTile;
                    const uint32_t b_addr = a_addr + q * kTChunk * kTKl;
#pragma unroll
                    for (uint32_t ks = 0; ks < kTKl / 32; ++ks)
                        t_mma_i8(tmem + l * kTChunk, t_desc_sw128(a_addr + 32 * ks),
                                 t_desc_sw128(b_addr + 32 * ks), ks);
                }
                t_commit(&sh.mma);
            }
            TP_MARK(3);  // MMA issue
            t_mbar_wait(&sh.mma, mma_phase);
            mma_phase ^= 1u;
            t_fence_after();
            TP_MARK(4);  // MMA completion
            // lane sums and the reference's tree for my row against the chunk,
            // kTSub columns at a time
            const uint32_t taddr = tmem + ((warp * 32u) << 16);
#pragma unroll 1
            for (uint32_t sc = 0; sc < kTChunk / kTSub; ++sc) {
                if (q * kTChunk + sc * kTSub >= nn) break;  // uniform: no new candidates left
                // lane l's exact integer sum for column jj, as a float
                auto lane_sum = [&](uint32_t l, uint32_t jj, uint32_t dot) {
                    const uint32_t j = q * kTChunk + sc * kTSub + jj;
                    const int32_t nb = M.nrm[j < kTMaxRows ? j : 0][l];
                    return float(na[l] + nb - 2 * int32_t(dot));
                };
                float h[kTSub], g2[kTSub];
                uint32_t v[32], w[32];
                // ((0+1)+(2+3)) + ((4+5)+(6+7)), two lanes' accumulators at a time
#pragma unroll
                for (uint32_t l = 0; l < 8; l += 2) {
                    t_ld32(taddr + l * kTChunk + sc * kTSub, v);
                    t_ld32(taddr + (l + 1) * kTChunk + sc * kTSub, w);
#pragma unroll
                    for (uint32_t jj = 0; jj < kTSub; ++jj) {
                        const float s2 =
                            __fadd_rn(lane_sum(l, jj, v[jj]), lane_sum(l + 1, jj, w[jj]));
                        if (l == 0) h[jj] = s2;
                        else if (l == 2) h[jj] = __fadd_rn(h[jj], s2);
                        else if (l == 4) g2[jj] = s2;
                        else g2[jj] = __fadd_rn(g2[jj], s2);
                    }
                }
                if (row_ok) {
#pragma unroll
                    for (uint32_t jj = 0; jj < kTSub; ++jj) {
                        const uint32_t j = q * kTChunk + sc * kTSub + jj;
                        if (j >= nn || !(i >= nn || j < i)) continue;
                        const uint32_t id_j = M.id[j];
                        // an id listed twice pairs with itself: try_insert
                        // ignores self (graph.hpp:116-129)
                        if (c.filter && id_j == id_i) continue;
                        const float d = __fadd_rn(h[jj], g2[jj]);
                        if (d < mx_i) {
                            const uint32_t pos = atomicAdd(&sh.cnt[i], 1u);
                            D[t_prow(i, nn, m) + 1 + pos] = pack_key(d, id_j);
                        }
                        if (d < M.mx[j]) {
                            const uint32_t pos = atomicAdd(&sh.cnt[j], 1u);
                            D[t_prow(j, nn, m) + 1 + pos] = pack_key(d, id_i);
                        }
                    }
                }
            }
            t_fence_before();
            __syncthreads();  // TMEM free for the next chunk's MMAs
        }
        TP_MARK(5);  // epilogue (TMEM loads, tree, proposals)
        __syncthreads();
        if (tid < m) D[t_prow(tid, nn, m)] = sh.cnt[tid];
        __syncthreads();  // buffer b and meta[b] are reused two nodes later
    }
    t_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                     "n"(kTTmemCols));
}

}  // namespace

#if KNNG_U8TC_PROF
extern "C" int knng_cuda_debug_u8tc_prof(unsigned long long* out) {
    if (cudaMemcpyFromSymbol(out, g_u8tc_prof, sizeof(unsigned long long) * 8) != cudaSuccess)
        return 1;
    const unsigned long long zero[8] = {};
    return cudaMemcpyToSymbol(g_u8tc_prof, zero, sizeof(zero)) != cudaSuccess;
}
#endif

bool u8_tc_supported(uint32_t stride, uint32_t cap) {
    return u8_lane_bytes(stride) == kTKl && 2 * cap <= kTMaxRows;
}

// The lane-major byte copy as a 2-D tensor (n rows x 8 Kl bytes) with a
// 128-byte box row and 128B swizzle, for gather4 (driver entry point, no
// libcuda link dependency).
bool u8_tc_make_map(const uint8_t* packed, uint32_t n, uint32_t stride, void* map_out) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const uint32_t kl = u8_lane_bytes(stride);
    cuuint64_t dims[2] = {cuuint64_t(8) * kl, n};
    cuuint64_t strides[1] = {cuuint64_t(8) * kl};
    cuuint32_t box[2] = {kTKl, 1};
    cuuint32_t es[2] = {1, 1};
    return enc(reinterpret_cast<CUtensorMap*>(map_out), CU_TENSOR_MAP_DATA_TYPE_UINT8, 2,
               const_cast<uint8_t*>(packed), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

void launch_join_u8_tc(const void* map, const CandView& c, IterCounters* ctr,
                       uint32_t max_active, const int32_t* lnorm, cudaStream_t s) {
    if (!max_active) return;
    static bool attr[kMaxDevices] = {};
    bool& done = attr[current_device()];
    if (!done) {
        check_launch(cudaFuncSetAttribute(join_u8_tc_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(kTSmem)));
        done = true;
    }
    uint32_t grid = device_sm_count();
    if (grid > max_active) grid = max_active;
    check_launch(cudaMemsetAsync(&ctr->work, 0, sizeof(uint32_t), s));
    join_u8_tc_kernel<<<grid, kTThreads, kTSmem, s>>>(*reinterpret_cast<const CUtensorMap*>(map),
                                                      c, ctr, lnorm);
}

}  // namespace knng_cuda
