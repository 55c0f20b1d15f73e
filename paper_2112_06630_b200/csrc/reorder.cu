// The locality reorder (reference reorder.hpp:22-50 greedy_cluster,
// dataset.hpp:237-245 apply_permutation, graph.hpp:150-166 KnnGraph::remap)
// as GPU kernels.
//
// Algorithm 1 of the paper is an inherently sequential walk (spot i+1 goes
// to the nearest unplaced neighbour of the node at spot i).  Its job is to
// put graph neighbours next to each other in memory; exactness of sigma is
// not part of the contract (only bijectivity and unchanged recall,
// acceptance.cpp:344-356, test_descent.cpp:211-224).  The
// parallel analogue here orders nodes by the single-linkage hierarchy of the
// current K-NN graph:
//   Boruvka rounds on the graph's edges: every component picks its lightest
//   outgoing edge (64-bit atomicMin on (distance bits, target)), components
//   hook along those edges (mutual pairs broken toward the smaller id) and
//   are flattened by pointer jumping; the component label of every node is
//   recorded after each round.
//   sigma = rank of each node under the lexicographic key
//   (label_R, label_{R-1}, ..., label_1, id), computed with R+1 stable LSD
//   radix passes (CUB).  Nodes merged early — the closest neighbours — end up
//   adjacent; whole clusters become contiguous ranges.
// apply_permutation is a row gather (one warp per row, 16-byte accesses) and
// remap renames ids and re-sorts each row (one warp per row).
#include <cub/device/device_radix_sort.cuh>

#include "kernels.cuh"

namespace knng_cuda {

namespace {

constexpr uint32_t kMaxRounds = 40;

__global__ void init_comp_kernel(uint32_t* comp, uint32_t n) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) comp[u] = u;
}

__global__ void reset_best_kernel(unsigned long long* best, uint32_t n) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) best[u] = ~0ull;
}

// lightest edge leaving each component
__global__ void min_edge_kernel(GraphView g, const uint32_t* comp, unsigned long long* best) {
    const size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= size_t(g.n) * g.k) return;
    const uint32_t u = uint32_t(e / g.k);
    const uint64_t key = g.keys[e];
    const uint32_t v = key_id(key);
    const uint32_t cu = comp[u], cv = comp[v];
    if (cu == cv) return;
    // (distance, target component) — ties resolve deterministically
    atomicMin(best + cu, (unsigned long long)((key & 0xffffffff00000000ull) | cv));
}

// hook each component root to the component its lightest edge reaches, only
// toward a smaller root id: parents strictly decrease, so the hook forest is
// acyclic even when ties make the lightest-edge graph cyclic (mutual lightest
// pairs hook the larger id under the smaller, as Boruvka does)
__global__ void hook_kernel(const uint32_t* comp, const unsigned long long* best,
                            uint32_t* parent, uint32_t n, uint32_t* merged) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n || comp[c] != c) return;
    const unsigned long long b = best[c];
    const uint32_t d = b == ~0ull ? c : uint32_t(b);
    parent[c] = d < c ? d : c;
    if (d < c) atomicAdd(merged, 1u);
}

__global__ void jump_kernel(const uint32_t* comp, uint32_t* parent, uint32_t n) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n || comp[c] != c) return;
    uint32_t r = parent[c];
    while (parent[r] != r) r = parent[r];
    parent[c] = r;
}

__global__ void relabel_kernel(uint32_t* comp, const uint32_t* parent, uint32_t* label_out,
                               uint32_t n) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const uint32_t r = parent[comp[u]];
    comp[u] = r;
    label_out[u] = r;
}

__global__ void gather_keys_kernel(const uint32_t* labels, const uint32_t* order,
                                   uint32_t* keys_out, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys_out[i] = labels[order[i]];
}

__global__ void invert_kernel(const uint32_t* order, uint32_t* sigma, uint32_t* sigma_inv,
                              uint32_t n) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const uint32_t u = order[p];
    sigma_inv[p] = u;
    sigma[u] = p;
}

// out.row(sigma[i]) = in.row(i)  (dataset.hpp:242-243), one warp per row
__global__ void permute_rows_kernel(const float* __restrict__ in, float* __restrict__ out,
                                    const uint32_t* __restrict__ sigma, uint32_t n,
                                    uint32_t stride) {
    const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= n) return;
    const uint32_t lane = lane_id();
    const float4* src = reinterpret_cast<const float4*>(in + size_t(i) * stride);
    float4* dst = reinterpret_cast<float4*>(out + size_t(sigma[i]) * stride);
    for (uint32_t c = lane; c < stride / 4; c += 32) dst[c] = __ldg(src + c);
    if ((stride & 3u) && lane < (stride & 3u)) {
        const uint32_t j = stride - (stride & 3u) + lane;
        out[size_t(sigma[i]) * stride + j] = in[size_t(i) * stride + j];
    }
}

// KnnGraph::remap (graph.hpp:150-166): row u -> row sigma[u], ids renamed;
// rows re-sorted by (distance, new id), flags and row maxima carried along.
__global__ void remap_kernel(GraphView in, GraphView out, const uint32_t* __restrict__ sigma) {
    const uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (u >= in.n) return;
    const uint32_t lane = lane_id(), k = in.k;
    const bool real = lane < k;
    const uint64_t key = real ? in.keys[size_t(u) * k + lane] : kEmptyKey;
    const uint32_t flag = (in.flags[u] >> lane) & 1u;
    const uint64_t nk = real ? ((key & 0xffffffff00000000ull) | sigma[key_id(key)]) : kEmptyKey;
    uint32_t rank = 0;
    for (uint32_t j = 0; j < k; ++j) {
        const uint64_t o = __shfl_sync(0xffffffffu, nk, j);
        rank += (o < nk) ? 1u : 0u;
    }
    const uint32_t dst_row = sigma[u];
    if (real) out.keys[size_t(dst_row) * k + rank] = nk;
    // flag bit moves with its entry: position `rank`
    uint32_t bits = 0;
    for (uint32_t j = 0; j < k; ++j) {
        const uint32_t rj = __shfl_sync(0xffffffffu, rank, j);
        const uint32_t fj = __shfl_sync(0xffffffffu, flag, j);
        bits |= fj << rj;
    }
    if (lane == 0) {
        out.flags[dst_row] = bits;
        out.maxd[dst_row] = in.maxd[u];
    }
}

inline uint32_t nblk(size_t items, uint32_t per) { return uint32_t((items + per - 1) / per); }

}  // namespace

// scratch layout: comp, parent, order_a, order_b, key_a, key_b (n u32 each),
// labels (kMaxRounds * n u32), best (n u64), merged (u32), cub temp.
size_t locality_permutation_scratch(uint32_t n) {
    size_t cub_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (const uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                    (uint32_t*)nullptr, int(n));
    // the same 256-byte rounding as launch_locality_permutation's carving
    auto r256 = [](size_t b) { return (b + 255) & ~size_t(255); };
    return 6 * r256(size_t(n) * 4) + r256(size_t(n) * 4 * kMaxRounds) + r256(size_t(n) * 8) + 256 +
           cub_bytes + 1024;
}

void launch_locality_permutation(const GraphView& g, uint32_t* sigma, uint32_t* sigma_inv,
                                 void* scratch, size_t scratch_bytes, cudaStream_t s) {
    const uint32_t n = g.n;
    char* p = static_cast<char*>(scratch);
    auto take = [&](size_t bytes) {
        char* r = p;
        p += (bytes + 255) & ~size_t(255);
        return r;
    };
    uint32_t* comp = reinterpret_cast<uint32_t*>(take(size_t(n) * 4));
    uint32_t* parent = reinterpret_cast<uint32_t*>(take(size_t(n) * 4));
    uint32_t* order_a = reinterpret_cast<uint32_t*>(take(size_t(n) * 4));
    uint32_t* order_b = reinterpret_cast<uint32_t*>(take(size_t(n) * 4));
    uint32_t* key_a = reinterpret_cast<uint32_t*>(take(size_t(n) * 4));
    uint32_t* key_b = reinterpret_cast<uint32_t*>(take(size_t(n) * 4));
    uint32_t* labels = reinterpret_cast<uint32_t*>(take(size_t(n) * 4 * kMaxRounds));
    unsigned long long* best = reinterpret_cast<unsigned long long*>(take(size_t(n) * 8));
    uint32_t* merged = reinterpret_cast<uint32_t*>(take(256));
    size_t cub_bytes = scratch_bytes - size_t(p - static_cast<char*>(scratch));
    void* cub_tmp = p;

    const uint32_t tb = 256;
    init_comp_kernel<<<nblk(n, tb), tb, 0, s>>>(comp, n);
    uint32_t rounds = 0, h_merged = 1;
    while (rounds < kMaxRounds && h_merged) {
        check_launch(cudaMemsetAsync(merged, 0, 4, s));
        reset_best_kernel<<<nblk(n, tb), tb, 0, s>>>(best, n);
        min_edge_kernel<<<nblk(size_t(n) * g.k, tb), tb, 0, s>>>(g, comp, best);
        hook_kernel<<<nblk(n, tb), tb, 0, s>>>(comp, best, parent, n, merged);
        jump_kernel<<<nblk(n, tb), tb, 0, s>>>(comp, parent, n);
        relabel_kernel<<<nblk(n, tb), tb, 0, s>>>(comp, parent, labels + size_t(rounds) * n, n);
        check_launch(cudaMemcpyAsync(&h_merged, merged, 4, cudaMemcpyDeviceToHost, s));
        check_launch(cudaStreamSynchronize(s), "locality permutation (Boruvka round)");
        ++rounds;
    }
    // LSD: stable sorts by label_1 .. label_R (last = most significant)
    init_comp_kernel<<<nblk(n, tb), tb, 0, s>>>(order_a, n);
    for (uint32_t r = 0; r < rounds; ++r) {
        gather_keys_kernel<<<nblk(n, tb), tb, 0, s>>>(labels + size_t(r) * n, order_a, key_a, n);
        size_t tmp = cub_bytes;
        check_launch(cub::DeviceRadixSort::SortPairs(cub_tmp, tmp, key_a, key_b, order_a, order_b,
                                                     int(n), 0, 32, s));
        std::swap(order_a, order_b);
    }
    invert_kernel<<<nblk(n, tb), tb, 0, s>>>(order_a, sigma, sigma_inv, n);
}

void launch_permute_rows(const float* in, float* out, const uint32_t* sigma, uint32_t n,
                         uint32_t stride, cudaStream_t s) {
    permute_rows_kernel<<<nblk(size_t(n) * 32, 256), 256, 0, s>>>(in, out, sigma, n, stride);
}

void launch_remap_graph(const GraphView& in, const GraphView& out, const uint32_t* sigma,
                        cudaStream_t s) {
    remap_kernel<<<nblk(size_t(in.n) * 32, 256), 256, 0, s>>>(in, out, sigma);
}

}  // namespace knng_cuda
