// Shared device helpers for the sm_100a NN-Descent kernels.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

namespace knng_cuda {

constexpr int kWarp = 32;
constexpr uint32_t kMaxK = 32;     // one warp lane per neighbour entry
constexpr uint32_t kMaxCap = 64;   // per-list candidate cap (2 ids per lane)
constexpr uint64_t kEmptyKey = ~0ull;

// A neighbour entry is one 64-bit key: float distance bits in the high word
// (distances are >= 0, so their bit patterns order like the values) and the
// id in the low word.  Ascending key order == (distance, id) order, the row
// order of KnnGraph::export_csv (graph.hpp:175-177).
__host__ __device__ __forceinline__ uint64_t pack_key(float dist, uint32_t id) {
#ifdef __CUDA_ARCH__
    return (uint64_t(__float_as_uint(dist)) << 32) | id;
#else
    uint32_t bits;
    __builtin_memcpy(&bits, &dist, 4);
    return (uint64_t(bits) << 32) | id;
#endif
}
__host__ __device__ __forceinline__ uint32_t key_id(uint64_t key) { return uint32_t(key); }
__device__ __forceinline__ float key_dist(uint64_t key) { return __uint_as_float(uint32_t(key >> 32)); }

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11): counter-based, so every edge/vertex
// draws from its own stream independent of launch order.
// ---------------------------------------------------------------------------
struct Philox4 {
    uint32_t x, y, z, w;
};

__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                                 uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return Philox4{c0, c1, c2, c3};
}

// Uniform integer in [0, range) from 32 random bits (multiply-shift; bias
// <= range / 2^32, immaterial for sampling).
__device__ __forceinline__ uint32_t bounded(uint32_t r, uint32_t range) {
    return __umulhi(r, range);
}

// ---------------------------------------------------------------------------
// Warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Bitonic sort of one 64-bit key per lane, ascending across the warp.
__device__ __forceinline__ uint64_t warp_sort_u64(uint64_t v) {
    const uint32_t lane = lane_id();
#pragma unroll
    for (uint32_t size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            const uint64_t other = __shfl_xor_sync(0xffffffffu, v, stride);
            const bool up = ((lane & size) == 0);
            const bool lower = ((lane & stride) == 0);
            const uint64_t lo = v < other ? v : other;
            const uint64_t hi = v < other ? other : v;
            v = (up == lower) ? lo : hi;
        }
    }
    return v;
}

// ---------------------------------------------------------------------------
// Per-device launch facts.  One process may drive several GPUs (the in-process
// multi-GPU driver), so kernel attributes, occupancy and SM counts are cached
// per device ordinal, never once per process.
// ---------------------------------------------------------------------------
constexpr int kMaxDevices = 64;

// A failed CUDA call inside a launch wrapper surfaces at once, as an exception
// the C-ABI guard (api.cu) turns into KNNG_CUDA_CUDA_ERROR with this message,
// instead of later under an unrelated call.
inline void check_launch(cudaError_t e, const char* what = "CUDA call in a launch wrapper",
                         const char* file = __builtin_FILE(), int line = __builtin_LINE()) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        const char* base = file;
        for (const char* q = file; *q; ++q)
            if (*q == '/') base = q + 1;
        throw std::runtime_error(std::string(what) + " (" + base + ":" + std::to_string(line) +
                                 "): " + cudaGetErrorString(e));
    }
}
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d & (kMaxDevices - 1);
}
inline uint32_t device_sm_count() {
    static uint32_t cache[kMaxDevices] = {};
    const int d = current_device();
    if (!cache[d]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
        cache[d] = v > 0 ? uint32_t(v) : 148u;
    }
    return cache[d];
}

// Coherent (L2) loads/stores for data shared across SMs under locks.
__device__ __forceinline__ uint64_t ld_cg_u64(const uint64_t* p) { return __ldcg(p); }
__device__ __forceinline__ uint32_t ld_cg_u32(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ float ld_cg_f32(const float* p) { return __ldcg(p); }
__device__ __forceinline__ void st_cg_u64(uint64_t* p, uint64_t v) { __stcg(p, v); }
__device__ __forceinline__ void st_cg_u32(uint32_t* p, uint32_t v) { __stcg(p, v); }
__device__ __forceinline__ void st_cg_f32(float* p, float v) { __stcg(p, v); }

}  // namespace knng_cuda
