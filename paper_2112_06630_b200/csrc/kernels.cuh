// Kernel-side views and launch wrappers shared by the host orchestrator.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace knng_cuda {

// The K-NN graph in HBM.  Per node u: k keys sorted ascending (see pack_key),
// a bitmask of is_new flags (bit i <-> key i), the cached row maximum used by
// the join's stale-upwards prefilter (descent.hpp:97-102), and a lock word.
struct GraphView {
    const float* data;  // n x stride, rows zero-padded to stride = ceil8(d)
    uint32_t n, k, stride;
    uint64_t* keys;     // n x k
    uint32_t* flags;    // n
    float* maxd;        // n
    uint32_t* locks;    // n
};

// Per-iteration candidate lists (CandidateSet layout, selection.hpp:22-49):
// per node 2*cap ids, new list first, old list second.
struct CandView {
    uint32_t cap;
    uint32_t* ids;      // n x 2cap
    uint32_t* raw_new;  // n, atomic append counters during sampling
    uint32_t* raw_old;  // n
    uint32_t* nc;       // n, final new counts
    uint32_t* oc;       // n, final old counts
};

// Device counters for one iteration.
struct IterCounters {
    unsigned long long changes;
    unsigned long long evals;
    unsigned long long cands;   // sum of (nn + no) over active nodes
    uint32_t active;            // number of nodes with nn > 0
    uint32_t pad;
};

// --- graph_kernels.cu ------------------------------------------------------
void launch_init_random(const GraphView& g, uint64_t seed, cudaStream_t s);
void launch_load_rows(const GraphView& g, const uint32_t* ids, const float* dists,
                      const uint8_t* flags, cudaStream_t s);
void launch_export_rows(const GraphView& g, uint32_t* ids, float* dists, uint8_t* flags,
                        cudaStream_t s);
void launch_indegree(const GraphView& g, uint32_t* indeg, cudaStream_t s);
void launch_sample(const GraphView& g, const CandView& c, const uint32_t* indeg, uint64_t seed,
                   cudaStream_t s);
void launch_finalize(const GraphView& g, const CandView& c, uint32_t* active,
                     IterCounters* ctr, cudaStream_t s);
void launch_reset_raw(const CandView& c, uint32_t n, cudaStream_t s);

// --- join.cu ---------------------------------------------------------------
// Local join of every active node (compute_step, descent.hpp:82-153).  The
// active count is read on the device from ctr->active (<= max_active).
void launch_join(const GraphView& g, const CandView& c, const uint32_t* active,
                 uint32_t max_active, IterCounters* ctr, cudaStream_t s);
// Distance stage only, writing each active node's D matrix to out + offsets[u].
void launch_join_distances(const GraphView& g, const CandView& c, const uint32_t* active,
                           uint32_t max_active, const uint64_t* offsets, float* out,
                           cudaStream_t s, IterCounters* ctr);
size_t join_smem_bytes(uint32_t cap);

// --- bruteforce.cu ---------------------------------------------------------
// Exact k nearest neighbours of the listed query rows among all n rows.
void launch_bruteforce_queries(const float* data, uint32_t n, uint32_t d, uint32_t stride,
                               uint32_t k, const uint32_t* queries, uint32_t nq,
                               uint64_t* scratch_top, uint32_t* out_ids, double* out_dists,
                               cudaStream_t s);
size_t bruteforce_scratch_keys(uint32_t nq);
void launch_iota(uint32_t* p, uint32_t n, cudaStream_t s);

// --- reorder.cu ------------------------------------------------------------
void launch_locality_permutation(const GraphView& g, uint32_t* sigma, uint32_t* sigma_inv,
                                 void* scratch, size_t scratch_bytes, cudaStream_t s);
size_t locality_permutation_scratch(uint32_t n);
void launch_permute_rows(const float* in, float* out, const uint32_t* sigma, uint32_t n,
                         uint32_t stride, cudaStream_t s);
void launch_remap_graph(const GraphView& in, const GraphView& out, const uint32_t* sigma,
                        cudaStream_t s);

}  // namespace knng_cuda
