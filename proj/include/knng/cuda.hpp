#pragma once
// knng::cuda — drop-in GPU replacement for knng::run (descent.hpp:193-255).
//
// Header-only C++ wrapper over the C-ABI of libknng_cuda.so (include/knng_cuda.h),
// placed where the reference keeps its own headers so a caller switches by
// changing `knng::run(data, params)` to `knng::cuda::run(data, params)`.  It
// takes and returns the reference's own types (Dataset, RunParams, RunResult,
// KnnGraph, Permutation) and throws the reference's exception types:
// std::invalid_argument for parameter errors (descent.hpp:29-35, 197), and
// std::runtime_error for device failures.  There is no CPU fallback.
//
// Build: add this repo's include/ and proj/include/ to the include path, link
// libknng_cuda.so.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "knng/descent.hpp"
#include "knng_cuda.h"

namespace knng::cuda {

namespace detail {

inline void check(int rc) {
    if (rc == KNNG_CUDA_OK) return;
    const std::string msg = knng_cuda_last_error();
    if (rc == KNNG_CUDA_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error("knng::cuda: " + msg);
}

// Dataset rows are padded to row_stride (dataset.hpp:61-77); the C-ABI takes
// the unpadded n x d matrix.
inline std::vector<float> unpadded(const Dataset& data) {
    std::vector<float> out(std::size_t(data.n()) * data.d());
    for (std::uint32_t i = 0; i < data.n(); ++i)
        std::memcpy(out.data() + std::size_t(i) * data.d(), data.row(i), sizeof(float) * data.d());
    return out;
}

}  // namespace detail

// knng::run on the GPU.  RunParams::strategy must be turbo and
// blocked_compute true (the reference defaults; naive/fused/flat are its
// benchmark baselines).  An observer makes the run read the graph back after
// every iteration (it stays on the device otherwise).  The returned graph is in
// original ids; its heap rows are rebuilt with KnnGraph::from_rows.
inline RunResult run(const Dataset& data, const RunParams& params,
                     const IterationObserver& observer = {}, int device = 0) {
    params.validate();
    if (data.n() <= params.k) throw std::invalid_argument("run: need n > k");
    if (params.strategy != SelectionStrategy::turbo || !params.blocked_compute)
        throw std::invalid_argument("knng::cuda::run: the GPU path implements turbo selection "
                                    "with the blocked join");

    knng_cuda_params p;
    knng_cuda_params_default(&p);
    p.k = params.k;
    p.max_candidates = params.max_candidates;
    p.termination_delta = params.termination_delta;
    p.max_iterations = params.max_iterations;
    p.reorder = params.reorder ? 1 : 0;
    p.reorder_after_iteration = params.reorder_after_iteration;
    p.seed = params.seed;
    p.device = device;
    // the observer sees a KnnGraph rebuilt from the device rows after every
    // iteration (descent.hpp:241), in the run's current labeling
    struct ObserverCtx {
        const IterationObserver* fn;
    } octx{&observer};
    if (observer) {
        p.observer = [](std::uint32_t it, std::uint32_t n_, std::uint32_t k_,
                        const std::uint32_t* ids_, const float* dists_, const std::uint8_t* fl_,
                        void* user) {
            std::vector<std::vector<NeighborEntry>> rows(n_, std::vector<NeighborEntry>(k_));
            for (std::uint32_t u = 0; u < n_; ++u)
                for (std::uint32_t i = 0; i < k_; ++i) {
                    const std::size_t q = std::size_t(u) * k_ + i;
                    rows[u][i] = NeighborEntry{ids_[q], dists_[q], fl_[q] != 0};
                }
            const KnnGraph g = KnnGraph::from_rows(k_, rows);
            (*static_cast<ObserverCtx*>(user)->fn)(it, g);
        };
        p.observer_user = &octx;
    }

    const std::uint32_t n = data.n(), k = params.k;
    const std::vector<float> rows = detail::unpadded(data);
    std::vector<std::uint32_t> ids(std::size_t(n) * k), sigma(params.reorder ? n : 0);
    std::vector<float> dists(std::size_t(n) * k);
    std::vector<std::uint8_t> flags(std::size_t(n) * k);
    std::vector<knng_cuda_iteration> its(params.max_iterations + 1);
    knng_cuda_metrics m{};
    m.iterations = its.data();
    m.capacity = static_cast<std::uint32_t>(its.size());
    detail::check(knng_cuda_run(rows.data(), n, data.d(), &p, ids.data(), dists.data(),
                                flags.data(), params.reorder ? sigma.data() : nullptr, &m));

    RunResult result;
    std::vector<std::vector<NeighborEntry>> graph_rows(n, std::vector<NeighborEntry>(k));
    for (std::uint32_t u = 0; u < n; ++u)
        for (std::uint32_t i = 0; i < k; ++i) {
            const std::size_t q = std::size_t(u) * k + i;
            graph_rows[u][i] = NeighborEntry{ids[q], dists[q], flags[q] != 0};
        }
    result.graph = KnnGraph::from_rows(k, graph_rows);
    for (std::uint32_t r = 0; r < m.n_rows && r < m.capacity; ++r)
        result.metrics.iterations.push_back(
            {its[r].iteration, its[r].wall_time_s, its[r].dist_evals, its[r].changes});
    result.metrics.total_wall_time_s = m.total_wall_time_s;
    result.metrics.total_dist_evals = m.total_dist_evals;
    result.metrics.total_changes = m.total_changes;
    if (params.reorder) {
        Permutation perm;
        perm.sigma = sigma;
        perm.sigma_inv.assign(n, 0);
        for (std::uint32_t i = 0; i < n; ++i) perm.sigma_inv[sigma[i]] = i;
        result.permutation = std::move(perm);
    }
    return result;
}

// The north-star signature: row-major float32 data, n, d, k, sample rate
// (max_candidates = lround(rho * k)), termination delta and seed in; n*k
// neighbour ids and squared distances out, rows sorted by (distance, id).
inline RunMetrics nndescent_l2(const float* data, std::uint32_t n, std::uint32_t d,
                               std::uint32_t k, double sample_rate, double delta,
                               std::uint64_t seed, std::uint32_t* out_ids, float* out_dists,
                               std::uint32_t max_iterations = 30) {
    std::vector<knng_cuda_iteration> its(max_iterations + 1);
    knng_cuda_metrics m{};
    m.iterations = its.data();
    m.capacity = static_cast<std::uint32_t>(its.size());
    detail::check(knng_cuda_nndescent_l2(data, n, d, k, sample_rate, delta, seed, max_iterations,
                                         1, out_ids, out_dists, &m));
    RunMetrics out;
    for (std::uint32_t r = 0; r < m.n_rows && r < m.capacity; ++r)
        out.iterations.push_back(
            {its[r].iteration, its[r].wall_time_s, its[r].dist_evals, its[r].changes});
    out.total_wall_time_s = m.total_wall_time_s;
    out.total_dist_evals = m.total_dist_evals;
    out.total_changes = m.total_changes;
    return out;
}

}  // namespace knng::cuda
