/*
 * knng_cuda.h — the C-ABI of libknng_cuda.so, the B200 (sm_100a) NN-Descent
 * K-NNG builder for squared L2.
 *
 * This is the drop-in boundary for the reference's one hot path, knng::run
 * (reference proj/include/knng/descent.hpp:193-255) and the pieces it is made
 * of.  The reference has no C-ABI of its own (it is a header-only C++
 * library); the entry points below are what its callers bind instead of the
 * C++ templates, each one citing the reference interface it replaces.  The
 * C++ drop-in wrapper with the reference's own types and exceptions is
 * proj/include/knng/cuda.hpp; Python binds the same symbols through ctypes
 * (paper_2112_06630_b200/_native.py).  See INTEGRATION.md.
 *
 * Conventions
 *  - Plain pointers and sizes only.  `data` is n x d row-major float32,
 *    unpadded (the library pads rows to ceil8(d) internally, as
 *    knng::Dataset does, dataset.hpp:61-77).
 *  - Entry points suffixed _device take DEVICE pointers and a cudaStream_t
 *    passed as void*; all others take HOST pointers and synchronise.
 *  - Neighbour rows are returned sorted ascending by (distance, id), the order
 *    of KnnGraph::export_csv (graph.hpp:169-184).  Rows passed IN may be in
 *    any order (e.g. the reference's heap order).
 *  - Return codes: KNNG_CUDA_OK or one of the errors below; a message for the
 *    calling thread is available from knng_cuda_last_error().  Parameter
 *    errors (KNNG_CUDA_INVALID_ARGUMENT) mirror the std::invalid_argument
 *    cases of the reference (descent.hpp:29-35,197; graph.hpp:37-38;
 *    dataset.hpp:74-75; selection.hpp:112-113).
 *  - No global mutable state besides cached device properties; calls from
 *    different host threads are independent.  There is no CPU fallback: with
 *    no usable CUDA device every compute entry point returns
 *    KNNG_CUDA_CUDA_ERROR.
 *  - Build limits (returned as KNNG_CUDA_INVALID_ARGUMENT): 2 <= k <= 32,
 *    k <= max_candidates <= 64, n < 2^31.
 */
#ifndef KNNG_CUDA_H
#define KNNG_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KNNG_CUDA_OK 0
#define KNNG_CUDA_INVALID_ARGUMENT 1
#define KNNG_CUDA_CUDA_ERROR 2
#define KNNG_CUDA_NCCL_ERROR 3
#define KNNG_CUDA_OUT_OF_MEMORY 4
#define KNNG_CUDA_NOT_IMPLEMENTED 5

#define KNNG_CUDA_MAX_K 32
#define KNNG_CUDA_MAX_CANDIDATES 64

/* knng::RunParams (descent.hpp:18-36).  strategy is always turbo and the
 * join always blocked (the reference defaults); naive/fused/flat are the
 * reference's benchmark baselines and are not part of this path. */
/* Per-iteration observer: knng::IterationObserver (descent.hpp:184, called at
 * :241) sees the graph after each iteration in the run's current internal
 * labeling (permuted ids after a reorder).  Called on the calling thread with
 * HOST arrays of n * k ids, squared distances and is_new flags, rows sorted by
 * (distance, id); setting it makes the run read the graph back every
 * iteration. */
typedef void (*knng_cuda_observer_fn)(uint32_t iteration, uint32_t n, uint32_t k,
                                      const uint32_t* ids, const float* dists,
                                      const uint8_t* flags, void* user);

typedef struct knng_cuda_params {
    uint32_t k;                        /* default 20 */
    uint32_t max_candidates;           /* default 50 (selection.hpp:15) */
    double termination_delta;          /* default 0.001 */
    uint32_t max_iterations;           /* default 30 */
    int32_t reorder;                   /* default 0 */
    uint32_t reorder_after_iteration;  /* default 1 */
    uint64_t seed;                     /* default 0 */
    int32_t device;                    /* CUDA device ordinal, default 0 */
    int32_t profile;                   /* 1: time each kernel with CUDA events */
    int32_t deterministic;             /* 1: seed-deterministic build (order-independent
                                          sampling and merges; default 0) */
    knng_cuda_observer_fn observer;    /* NULL (default): none */
    void* observer_user;               /* passed back to observer */
} knng_cuda_params;

/* knng::IterationMetrics (descent.hpp:38-43).  `changes` counts successful
 * bounded inserts like KnnGraph::changes_ (graph.hpp:126); inserts are applied
 * concurrently, so early-iteration counts differ from the sequential
 * reference's while agreeing near the termination threshold. */
typedef struct knng_cuda_iteration {
    uint32_t iteration;  /* 0 = random initialisation */
    double wall_time_s;
    uint64_t dist_evals;
    uint64_t changes;
    uint64_t join_candidates;  /* sum of (nn_u + no_u) over the iteration's joins */
    double join_ms;            /* distance-kernel device time (params.profile only) */
} knng_cuda_iteration;

/* Per-kernel device time (CUDA events on the library's stream), filled when
 * params.profile != 0.  Index with the KNNG_CUDA_KERNEL_* constants. */
#define KNNG_CUDA_KERNEL_INIT 0      /* init_random */
#define KNNG_CUDA_KERNEL_DEGREE 1    /* in-degree histogram */
#define KNNG_CUDA_KERNEL_SAMPLE 2    /* turbo offers */
#define KNNG_CUDA_KERNEL_FINALIZE 3  /* dedup, flag_consumed, join bookkeeping */
#define KNNG_CUDA_KERNEL_JOIN 4      /* local-join distance kernel */
#define KNNG_CUDA_KERNEL_REORDER 5   /* locality permutation + gathers */
#define KNNG_CUDA_KERNEL_MERGE 6     /* bounded sorted-list updates */
#define KNNG_CUDA_KERNEL_INDEX 7     /* block offsets + reverse index */
#define KNNG_CUDA_KERNEL_COUNT 8

/* knng::RunMetrics (descent.hpp:45-68) plus device-side accounting.  The
 * caller provides `iterations` with room for `capacity` rows
 * (max_iterations + 1 suffices). */
typedef struct knng_cuda_metrics {
    knng_cuda_iteration* iterations;
    uint32_t capacity;
    uint32_t n_rows;                 /* rows written (iteration 0 included) */
    double total_wall_time_s;
    uint64_t total_dist_evals;
    uint64_t total_changes;
    double kernel_ms[KNNG_CUDA_KERNEL_COUNT];
    uint64_t kernel_launches[KNNG_CUDA_KERNEL_COUNT];
    uint64_t join_candidates;        /* sum over joins of (nn_u + no_u) */
    uint64_t join_evals;             /* distance evaluations inside the join kernel */
    uint64_t h2d_bytes;              /* host->device bytes moved by the call */
    uint64_t d2h_bytes;              /* device->host bytes moved by the call */
} knng_cuda_metrics;

/* Fills *p with the reference defaults (descent.hpp:18-28). */
void knng_cuda_params_default(knng_cuda_params* p);

/* Thread-local message for the last failing call on this thread. */
const char* knng_cuda_last_error(void);

/* Number of visible CUDA devices (0 when none). */
int knng_cuda_device_count(void);

/*
 * The north-star entry point: replaces knng::run(Dataset, RunParams)
 * (descent.hpp:193-255) for squared L2.  HOST pointers.
 *   sample_rate rho -> max_candidates = lround(rho * k) (PAPER.md:88,
 *   SPEC.md:266,308); must be >= k.  out_ids/out_dists: n*k each, rows
 *   sorted by (distance, id).  out_metrics may be NULL.  num_gpus > 1 runs
 *   the vertex-sharded build over that many GPUs in this process
 *   (knng_cuda_run_multi, shard r on device r % device count).
 */
int knng_cuda_nndescent_l2(const float* data, uint32_t n, uint32_t d, uint32_t k,
                           double sample_rate, double delta, uint64_t seed,
                           uint32_t max_iterations, int num_gpus, uint32_t* out_ids,
                           float* out_dists, knng_cuda_metrics* out_metrics);

/* knng::run with full RunParams.  HOST pointers; out_flags (n*k, 1 = is_new)
 * and out_metrics may be NULL.  out_sigma (n, nullable) receives the
 * locality permutation when params->reorder is set. */
int knng_cuda_run(const float* data, uint32_t n, uint32_t d, const knng_cuda_params* params,
                  uint32_t* out_ids, float* out_dists, uint8_t* out_flags,
                  uint32_t* out_sigma, knng_cuda_metrics* out_metrics);

/* Same, DEVICE pointers (data: n*d floats; out_ids/out_dists: n*k) on the
 * given stream (void* = cudaStream_t, NULL = a library stream). */
int knng_cuda_run_device(const float* d_data, uint32_t n, uint32_t d,
                         const knng_cuda_params* params, uint32_t* d_out_ids,
                         float* d_out_dists, knng_cuda_metrics* out_metrics, void* stream);

/*
 * One local join from a fixed state — the parity entry.  Replaces
 * knng::compute_step(KnnGraph&, const CandidateSet&, const Dataset&,
 * EvalCounter&) (descent.hpp:82-153) applied to
 * KnnGraph::from_rows(k, rows) (graph.hpp:70-93).
 *   in_ids/in_dists/in_flags: n*k graph rows (any order, e.g. heap order);
 *   cand_ids: n*2*cap, per node `new` block then `old` block
 *   (CandidateSet layout, selection.hpp:22-49); new_counts/old_counts: n.
 *   Outputs (n*k, rows sorted by (distance,id)): ids, dists, is_new flags;
 *   out_rev_deg (n): k + in-degree (KnnGraph::reverse_degree, graph.hpp:98);
 *   changes: successful inserts; evals: distance evaluations.
 */
int knng_cuda_local_join(const float* data, uint32_t n, uint32_t d, uint32_t k, uint32_t cap,
                         const uint32_t* in_ids, const float* in_dists, const uint8_t* in_flags,
                         const uint32_t* cand_ids, const uint32_t* new_counts,
                         const uint32_t* old_counts, uint32_t* out_ids, float* out_dists,
                         uint8_t* out_flags, uint32_t* out_rev_deg, uint64_t* changes,
                         uint64_t* evals, int device);

/* The join's distance stage alone, for per-pair bit-exactness checks against
 * mutual_block_distances / block_l2_sq (distance.hpp:134-190) as driven by
 * compute_step.  For every node u with new_counts[u] > 0 writes the
 * (new_counts[u]) x (new_counts[u] + old_counts[u]) matrix D_u, row i = new
 * candidate i, column j = new candidate j (j < nn) or old candidate j - nn,
 * into out_dists + offsets[u] (row-major; entries of the new x new block with
 * j <= i are left untouched).  offsets: n entries, computed by the caller. */
int knng_cuda_candidate_distances(const float* data, uint32_t n, uint32_t d, uint32_t cap,
                                  const uint32_t* cand_ids, const uint32_t* new_counts,
                                  const uint32_t* old_counts, const uint64_t* offsets,
                                  float* out_dists, uint64_t total, int device);

/* KnnGraph::init_random (graph.hpp:34-67): k distinct uniform ids != u per
 * node (counter-based Philox draws, not the reference's sequential
 * mt19937_64 stream) with their true distances.  Rows sorted by (dist,id). */
int knng_cuda_init_random(const float* data, uint32_t n, uint32_t d, uint32_t k, uint64_t seed,
                          uint32_t* out_ids, float* out_dists, uint8_t* out_flags,
                          uint32_t* out_rev_deg, uint64_t* evals, int device);

/* select_turbo (selection.hpp:282-320) followed by flag_consumed for every
 * node (descent.hpp:225, graph.hpp:133-143).  Same sampling law (offer each
 * edge endpoint to the other with probability min(1, cap/deg), dedup across
 * both lists, bounded lists), applied concurrently with Philox draws.
 * out_flags_after: n*k flags in the caller's entry order after consumption. */
int knng_cuda_select(uint32_t n, uint32_t k, uint32_t cap, const uint32_t* in_ids,
                     const float* in_dists, const uint8_t* in_flags, uint64_t seed,
                     uint32_t* cand_ids, uint32_t* new_counts, uint32_t* old_counts,
                     uint8_t* out_flags_after, int device);

/* brute_force_knng (oracle.hpp:92-127) on the GPU: exact k nearest
 * neighbours, rows sorted by (distance, id) with distances evaluated in
 * float64 like l2_sq_double (oracle.hpp:50-66).  No size guard. */
int knng_cuda_bruteforce_knng(const float* data, uint32_t n, uint32_t d, uint32_t k,
                              uint32_t* out_ids, double* out_dists, int device);

/* The same for a subset of query rows (nq ids in `queries`; NULL = all n):
 * row i of the outputs is the exact k-NN of node queries[i] among all n
 * nodes.  Used to measure recall on a sample of nodes at large n. */
int knng_cuda_bruteforce_queries(const float* data, uint32_t n, uint32_t d, uint32_t k,
                                 const uint32_t* queries, uint32_t nq, uint32_t* out_ids,
                                 double* out_dists, int device);

/* greedy_cluster's role (reorder.hpp:22-50) on the GPU: a locality
 * permutation built from the current graph (sigma[u] = new position of u,
 * sigma_inv[p] = node at position p).  A parallel analogue, not Algorithm 1's
 * exact sequential walk. */
int knng_cuda_locality_permutation(uint32_t n, uint32_t k, const uint32_t* ids,
                                   const float* dists, uint32_t* sigma, uint32_t* sigma_inv,
                                   int device);

/*
 * Multi-GPU shards — vertex-range ownership with the data
 * replicated.  Shard r owns rows [r*chunk, min(n, (r+1)*chunk)): their graph
 * rows, candidate lists, joins and merges; only the row maxima (n floats, the
 * join prefilter's bound) are replicated.  Replaces the reference loop
 * descent.hpp:219-243 with, per iteration:
 *   knng_cuda_shard_degree   partial in-degree of the owned rows' edges into
 *                            info.indeg;           caller: all-reduce (sum, n u32)
 *   knng_cuda_shard_sample   turbo sampling over the owned rows' edges (local
 *                            offers applied; accepted reverse offers for rows
 *                            owned elsewhere grouped by owner);
 *                                                  caller: all-to-all (4 u32 each)
 *   knng_cuda_shard_offers   received offers into the owned lists
 *   knng_cuda_shard_step     finalize, local join of the owned active nodes,
 *                            merges into owned rows, pre-reduced proposal
 *                            records (target, id, dist bits) for rows owned
 *                            elsewhere (<= k per target);
 *                                                  caller: all-to-all (3 u32 each)
 *   knng_cuda_shard_merge    received records into owned rows;
 *                                                  caller: all-gather of the owned
 *                                                  slices of info.maxd, all-reduce
 *                                                  of changes (termination test)
 * Work is stream-ordered on info.stream: the caller's stream when one is
 * given (cudaStreamLegacy = (void*)1 for the default stream), else a stream
 * of the shard's own; sample, step and merge return host counts and so
 * synchronise it.
 * knng_cuda_run_multi drives the same phases for N GPUs in one process.
 * Deterministic mode is not supported on shards.
 */
typedef struct knng_cuda_shard knng_cuda_shard;

typedef struct knng_cuda_shard_info {
    uint64_t* keys;       /* rows_alloc x k (owned rows valid): (dist bits << 32) | id */
    uint32_t* flags;      /* rows_alloc: bit i = entry i is new */
    float* maxd;          /* rows_alloc: row maximum, every row (replicated) */
    uint32_t* indeg;      /* n: in-degree (partial after shard_degree; the sum after
                             the caller's all-reduce) */
    uint32_t rows_alloc;  /* nranks * chunk (>= n), so every rank's slice is `chunk` rows */
    uint32_t chunk;
    uint32_t lo, hi;      /* owned rows */
    void* stream;         /* cudaStream_t of the shard's work */
    uint64_t seg_cap;     /* offer records per destination segment of shard_sample */
} knng_cuda_shard_info;

int knng_cuda_shard_create(const float* d_data, uint32_t n, uint32_t d,
                           const knng_cuda_params* params, uint32_t rank, uint32_t nranks,
                           void* stream, knng_cuda_shard** out, knng_cuda_shard_info* info);
int knng_cuda_shard_destroy(knng_cuda_shard* shard);
/* The run's seeds: std::mt19937_64(seed) outputs, [0] init, [i] iteration i
 * (descent.hpp:201-221) — identical to the single-GPU path. */
void knng_cuda_seed_sequence(uint64_t seed, uint32_t count, uint64_t* out);
/* init_random (graph.hpp:34-67) of the owned rows; per-node Philox draws, so
 * the initial graph does not depend on the number of ranks. */
int knng_cuda_shard_init(knng_cuda_shard* shard, uint64_t seed);
int knng_cuda_shard_degree(knng_cuda_shard* shard);
/* select_turbo (selection.hpp:282-320) over the owned edges with iteration
 * seed `seed`.  send_counts: nranks offer counts; segment r of
 * *send_records starts at record r * info.seg_cap (4 u32 per record). */
int knng_cuda_shard_sample(knng_cuda_shard* shard, uint64_t seed, uint64_t* send_counts,
                           const uint32_t** send_records);
int knng_cuda_shard_offers(knng_cuda_shard* shard, const uint32_t* d_records, uint64_t count);
/* counters: [0] distance evaluations, [1] candidates joined, [2] inserts into
 * owned rows so far, [3] active nodes.  send_counts: nranks record counts;
 * *send_records: device pointer to 3 * sum(send_counts) u32, grouped by owner
 * in rank order. */
int knng_cuda_shard_step(knng_cuda_shard* shard, uint64_t* counters, uint64_t* send_counts,
                         const uint32_t** send_records);
/* d_records: count records (3 u32 each) for owned targets; *changes = all
 * inserts into owned rows this iteration (local + received). */
int knng_cuda_shard_merge(knng_cuda_shard* shard, const uint32_t* d_records, uint64_t count,
                          uint64_t* changes);
/* owned rows, sorted by (distance, id): (hi - lo) x k ids and distances. */
int knng_cuda_shard_export(knng_cuda_shard* shard, uint32_t* d_ids, float* d_dists);
/* The locality reorder on shards (descent.hpp:230-235), after iteration
 * params.reorder_after_iteration: the caller first all-gathers every shard's
 * owned rows (info.keys rows [lo, hi) x k, info.flags, info.maxd) into every
 * shard; each shard then computes sigma from the whole graph (a deterministic
 * function of it, so every shard gets the same one) and permutes its data
 * and graph.  Shards go on owning rows [lo, hi) of the permuted order, i.e.
 * contiguous ranges of sigma.  *info is refreshed (the graph buffers move);
 * *d_sigma / *d_sigma_inv (n u32, device) map the exported rows back
 * (descent.hpp:245). */
int knng_cuda_shard_reorder(knng_cuda_shard* shard, knng_cuda_shard_info* info,
                            const uint32_t** d_sigma, const uint32_t** d_sigma_inv);
/* This shard's share so far: per-kernel device times (params.profile at
 * creation) and one row per iteration (its evaluations, candidates, inserts
 * into owned rows and join-kernel time). */
int knng_cuda_shard_metrics(knng_cuda_shard* shard, knng_cuda_metrics* out);

/* knng::run (descent.hpp:193-255) over num_gpus shards in ONE process, shard r
 * on device devices[r] (NULL: r % device count; several shards may share a
 * device).  The exchanges are peer copies between the shards' streams
 * (NVLink / NVSwitch between GPUs).  Host data in, host graph out (n x k,
 * rows sorted by (distance, id)); metrics as knng_cuda_run.  params.reorder
 * and params.deterministic are not supported here (KNNG_CUDA_NOT_IMPLEMENTED). */
int knng_cuda_run_multi(const float* data, uint32_t n, uint32_t d, const knng_cuda_params* params,
                        int num_gpus, const int* devices, uint32_t* out_ids, float* out_dists,
                        knng_cuda_metrics* out_metrics);

#ifdef __cplusplus
}
#endif

#endif /* KNNG_CUDA_H */
