// Kernel-side views and launch wrappers shared by the host orchestrator.
#pragma once

#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "common.cuh"

namespace knng_cuda {

// The K-NN graph in HBM.  Per node u: k keys sorted ascending (see pack_key),
// a bitmask of is_new flags (bit i <-> key i), and the cached row maximum
// (the reference's row_max_, graph.hpp:216-221).
struct GraphView {
    const float* data;  // n x stride, rows zero-padded to stride = ceil8(d)
    uint32_t n, k, stride;
    uint64_t* keys;     // n x k
    uint32_t* flags;    // n
    float* maxd;        // n
    // Rows this device owns (multi-GPU sharding): init, finalize,
    // the join's active nodes and the merges cover [lo, hi); the graph itself
    // is replicated (allgathered each iteration).  Single GPU: [0, n).
    uint32_t lo, hi;
};

// Per-iteration candidate lists (CandidateSet layout, selection.hpp:22-49):
// per node 2*cap ids, new list first, old list second; plus the join's
// bookkeeping: the size and offset of each active node's proposal block, and
// the reverse index (for every candidate t, where t's row of each proposal
// block naming t starts) that lets one warp per target pull its proposals.
struct CandView {
    uint32_t cap;
    uint32_t* ids;       // n x 2cap
    uint32_t* raw_new;   // n, atomic append counters during sampling
    uint32_t* raw_old;   // n
    uint32_t* nc;        // n, final new counts
    uint32_t* oc;        // n, final old counts
    uint64_t* dsz;       // n, words in u's proposal block (0 when nn == 0)
    uint64_t* doff;      // n, exclusive prefix sum of dsz
    uint32_t* revcnt;    // n, how many active lists name t
    uint32_t* roff;      // n, exclusive prefix sum of revcnt
    uint32_t* rcur;      // n, scatter cursors
    uint64_t* rev;       // total entries: word offset in D of t's row of u's proposal block
    uint64_t* D;         // proposal blocks, see join.cu
    int filter;          // 1: keep only proposals below the target's row maximum
    float* cmax;         // n x 2cap, the row maximum of each listed candidate
                         // (iteration start), beside ids
    uint4* arec;         // per active index: {u, nn | no << 16, doff lo, doff hi}
    uint32_t* hubs;      // n: targets with more than kHubEntries reverse entries
    // deterministic mode (knng_cuda_params.deterministic): sampling appends
    // every accepted offer, as a key (pair weight << 32 | id), to n x 4cap
    // raw lists (new 2cap, old 2cap; no reservoir); a list that received more
    // than 2cap offers is rebuilt from all of them as the 2cap smallest keys
    // (det_fix_*: order-free); finalize keeps the cap offers of smallest pair
    // weight, and the merges keep the smaller copy of a present id and count
    // changes as |final row \ initial row|
    unsigned long long* raw;
    int det;
    // in-degree kept up to date by the merges (single-GPU builds, counters
    // in per-iteration slots): a merge that changes row t adds 1 for each id
    // that came in and subtracts 1 for each id that left, unless the next
    // iteration recounts (next slot's recount flag).  nullptr: recounted by
    // indegree_kernel every iteration
    uint32_t* indeg_inc;
};

// Device counters for one iteration.
struct IterCounters {
    unsigned long long changes;
    unsigned long long evals;
    unsigned long long cands;    // sum of (nn + no) over active nodes
    unsigned long long dwords;   // total distance-block words (u64)
    unsigned long long rev;      // total reverse-index entries
    uint32_t active;             // number of nodes with nn > 0
    uint32_t work;               // dynamic work counter
    uint32_t overflow;           // distance blocks exceed the buffer: join skipped
    uint32_t hubs;               // merge: targets left to the per-CTA hub merge
    uint32_t work2;              // second work counter (byte-valued join: staged nodes)
    uint32_t halt;               // set by iter_end_kernel: an earlier iteration met the
                                 // termination test (or overflowed); this one is a no-op
    uint32_t recount;            // this iteration's selection recounts the in-degree; the
                                 // previous iteration's merges then skip their updates
    unsigned long long screened;   // screened join: pairs bounded
    unsigned long long survivors;  // screened join: pairs evaluated exactly
    uint32_t det_ovf;              // deterministic sampling: some raw list overflowed 2cap
    uint32_t pad_;
};

// --- graph_kernels.cu ------------------------------------------------------
// packed / lnorm: byte-valued data's lane-major copy (join_u8.cu); distances
// then come from exact integer lane sums (bit-identical to the FP32 path)
void launch_init_random(const GraphView& g, uint64_t seed, cudaStream_t s,
                        const uint8_t* packed = nullptr, const int32_t* lnorm = nullptr);
void launch_load_rows(const GraphView& g, const uint32_t* ids, const float* dists,
                      const uint8_t* flags, cudaStream_t s);
void launch_export_rows(const GraphView& g, uint32_t* ids, float* dists, uint8_t* flags,
                        cudaStream_t s);
// gate (optional): the iteration's counters; the kernel does nothing when
// gate->halt is set (iterations enqueued past termination, see run_engine)
void launch_indegree(const GraphView& g, uint32_t* indeg, cudaStream_t s,
                     const IterCounters* gate = nullptr);
// gate: the iteration's counters (halt flag; det_ovf, set when a deterministic
// raw list overflows).  det_seed keys the deterministic pair weights (the
// iteration seed, the same value finalize_det gets).
void launch_sample(const GraphView& g, const CandView& c, const uint32_t* indeg, uint64_t seed,
                   cudaStream_t s, IterCounters* gate, uint64_t det_seed);
// Partitioned selection (multi-GPU): the owned rows' edges only.  Partial
// in-degree (the caller all-reduces it); sampling with local offers applied
// and accepted remote reverse offers appended as {target, cand, is_new, slot
// draw} to the owner's segment of send (nranks x seg_cap, counts in dst_cnt);
// received offers inserted by launch_apply_offers.
void launch_indegree_owned(const GraphView& g, uint32_t* indeg, cudaStream_t s);
void launch_sample_owned(const GraphView& g, const CandView& c, const uint32_t* indeg,
                         uint64_t seed, const IterCounters* gate, uint32_t chunk,
                         uint32_t nranks, uint32_t* dst_cnt, uint4* send, uint64_t seg_cap,
                         cudaStream_t s);
void launch_apply_offers(const CandView& c, const uint4* recs, uint64_t count,
                         const IterCounters* gate, cudaStream_t s);
// dedup + flag_consumed + join bookkeeping (active list, block sizes, reverse counts)
void launch_finalize(const GraphView& g, const CandView& c, uint32_t* active,
                     IterCounters* ctr, cudaStream_t s, uint64_t seed = 0);
// join bookkeeping only, for externally supplied candidate lists (fixed-state entries)
void launch_bookkeeping(const GraphView& g, const CandView& c, uint32_t* active,
                        IterCounters* ctr, cudaStream_t s);
void launch_reset_raw(const CandView& c, uint32_t n, cudaStream_t s,
                      const IterCounters* gate = nullptr);
// next->halt = cur->halt | cur->overflow | (changes < threshold): the device-side
// termination test (descent.hpp:242) that gates the iterations enqueued after cur;
// next[1].recount = cur->changes > recount_above (the iteration after next
// recounts the in-degree when this one changed many rows: the incremental
// updates would cost more atomics than the recount)
void launch_iter_end(const IterCounters* cur, IterCounters* next, double threshold,
                     double recount_above, cudaStream_t s);
// in-degree recount gated on gate->recount (and not halted)
void launch_indegree_gated(const GraphView& g, uint32_t* indeg, const IterCounters* gate,
                           cudaStream_t s);

// --- join.cu ---------------------------------------------------------------
// Exclusive scans dsz -> doff and revcnt -> roff (CUB); scratch sizing.
size_t join_scan_scratch(uint32_t n);
void launch_join_offsets(const CandView& c, uint32_t n, uint32_t lo, uint32_t hi, void* scratch,
                         size_t scratch_bytes,
                         cudaStream_t s);
// Sets ctr->overflow when the distance blocks need more than `capacity` floats
// (the join stages then return at once; the host grows the buffer and
// relaunches them), so an iteration needs no host round trip before its join.
void launch_check_capacity(IterCounters* ctr, unsigned long long capacity, cudaStream_t s);
// Reverse index scatter (one warp per active node).
void launch_scatter_rev(const CandView& c, const uint32_t* active, IterCounters* ctr,
                        uint32_t max_active, uint32_t n, cudaStream_t s);
// Distance stage of the local join: every active node's distance block.
void launch_join_distances(const GraphView& g, const CandView& c, const uint32_t* active,
                           IterCounters* ctr, uint32_t max_active, cudaStream_t s);
// --- join5.cu ----------------------------------------------------------------
// The same distance stage with 5 x 10 tiles aligned to the reference's
// 5-blocking (same proposal blocks, bit-identical distances).
void launch_join5(const GraphView& g, const CandView& c, IterCounters* ctr, uint32_t max_active,
                  cudaStream_t s);
// --- join_gl.cu --------------------------------------------------------------
// Long rows: the distance stage with candidate rows loaded straight into
// registers from a lane-major copy of the data (same proposal blocks,
// bit-identical distances).  gl_row_floats: floats per row of that copy,
// which holds n + 1 rows (row n all zero).
uint32_t gl_row_floats(uint32_t stride);
void launch_gl_pack(const float* data, uint32_t n, uint32_t stride, float* dl, cudaStream_t s);
void launch_join_gl(const CandView& c, const float* dl, uint32_t n, uint32_t stride,
                    IterCounters* ctr, uint32_t max_active, cudaStream_t s);
// --- join_tc.cu --------------------------------------------------------------
// ||x||^2 (rounded down) and ||x|| (rounded up) of every data row.
void launch_row_norms(const float* data, uint32_t n, uint32_t stride, float* nrm2, float* nrmu,
                      cudaStream_t s);
// Distance stage screened on the tensor cores: same proposal blocks as
// launch_join_distances with the prefilter on (see join_tc.cu).  Nodes too
// large for its shared-memory arena are listed in ovf (count in octr->active)
// and run through launch_join_distances.
void launch_join_tc(const GraphView& g, const CandView& c, IterCounters* ctr, uint32_t max_active,
                    const float* nrm2, const float* nrmu, uint4* ovf, IterCounters* octr,
                    cudaStream_t s);
// --- join_u8.cu --------------------------------------------------------------
// Byte-valued data (every coordinate an integer in [0, 255], stride / 8 <= 258):
// the distance stage on the integer tensor cores, bit-identical to the FP32
// tile kernel.  u8_eligible checks the data on the device (one host sync).
uint32_t u8_lane_bytes(uint32_t stride);  // Kl: bytes per reference lane per row
bool u8_eligible(const float* data, uint32_t n, uint32_t stride, uint32_t* d_flag,
                 cudaStream_t s);
void launch_u8_pack(const float* data, uint32_t n, uint32_t stride, uint8_t* packed,
                    int32_t* lnorm, cudaStream_t s);
void launch_join_u8(const GraphView& g, const CandView& c, IterCounters* ctr, uint32_t max_active,
                    const uint8_t* packed, const int32_t* lnorm, cudaStream_t s);
// --- join_u8_tc.cu -----------------------------------------------------------
// The byte-valued join on tcgen05 (TMA gather4 -> SMEM -> kind::i8 MMA -> TMEM),
// bit-identical to launch_join_u8.  Supported for Kl = 128 and cap <= 52; the
// tensor map (CUtensorMap, 128 bytes) describes the lane-major byte copy.
bool u8_tc_supported(uint32_t stride, uint32_t cap);
bool u8_tc_make_map(const uint8_t* packed, uint32_t n, uint32_t stride, void* map_out);
void launch_join_u8_tc(const void* map, const CandView& c, IterCounters* ctr,
                       uint32_t max_active, const int32_t* lnorm, cudaStream_t s);
// Update stage: one warp per target pulls and merges its proposals.
void launch_join_merge(const GraphView& g, const CandView& c, IterCounters* ctr,
                       cudaStream_t s);
// Multi-GPU: records (t, id, dist bits) for non-owned targets; pass 1 counts
// per target (counts[n]), pass 2 writes at offsets[t] (exclusive scan).
void launch_export_remote(const GraphView& g, const CandView& c, IterCounters* ctr,
                          uint32_t* counts, const uint64_t* offsets, uint32_t* records,
                          bool write, cudaStream_t s);
// Multi-GPU: merge received records into the owned rows (counting sort by
// target, then one warp per owned target).
void launch_merge_received(const GraphView& g, const uint32_t* records, uint64_t count,
                           uint32_t* cnt, uint32_t* off, uint32_t* cur, uint64_t* grouped,
                           void* scratch, size_t scratch_bytes, IterCounters* ctr,
                           cudaStream_t s);

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

// --- host_io.cu -----------------------------------------------------------
// One host buffer <-> one device buffer of `bytes` bytes.
struct HostSeg {
    void* host;
    void* dev;
    size_t bytes;
};
bool host_is_pinned(const void* p);
// Pageable buffers go through a pinned ring drained / filled by host threads
// while the copy engine runs; pinned ones are copied directly.
// copy_from_host returns once the host buffers may be reused (copies
// enqueued on s); copy_to_host returns once the data is in the host buffers.
void copy_from_host(const std::vector<HostSeg>& segs, cudaStream_t s);
void copy_to_host(const std::vector<HostSeg>& segs, cudaStream_t s);

}  // namespace knng_cuda
