// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A thin extern "C" harness around the UNMODIFIED reference headers
// (/root/reference/proj/include/knng/*.hpp, included read-only, nothing copied).
// Built by oracle/Makefile into oracle/_ref/libknng_ref.so.  The Python test
// suite and bench.py's `--impl reference` / cpu_baseline leg call it through
// ctypes; it is the strongest available oracle: the reference's own code.
//
// Conventions: input data is n x d row-major float32 (unpadded); the harness
// builds a knng::Dataset (which pads rows to ceil8(d), dataset.hpp:61-77).
// Graph rows are exported in the reference's internal HEAP order
// (graph.hpp:17-21, 28-222) as parallel ids / dists / flags arrays.
// Every function returns 0 on success, 1 on std::invalid_argument, 2 on any
// other exception; the message is available from ref_last_error().

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "knng/knng.hpp"

using namespace knng;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

Dataset make_dataset(const float* data, std::uint32_t n, std::uint32_t d) {
    Dataset ds(n, d);
    for (std::uint32_t i = 0; i < n; ++i)
        std::memcpy(ds.row(i), data + std::size_t(i) * d, sizeof(float) * d);
    return ds;
}

void export_graph(const KnnGraph& g, std::uint32_t* ids, float* dists, std::uint8_t* flags,
                  std::uint32_t* rev_deg) {
    const std::uint32_t n = g.n(), k = g.k();
    for (std::uint32_t u = 0; u < n; ++u) {
        for (std::uint32_t i = 0; i < k; ++i) {
            const NeighborEntry& e = g.entry(u, i);
            const std::size_t p = std::size_t(u) * k + i;
            if (ids) ids[p] = e.id;
            if (dists) dists[p] = e.dist;
            if (flags) flags[p] = e.is_new ? 1 : 0;
        }
        if (rev_deg) rev_deg[u] = g.reverse_degree(u);
    }
}

KnnGraph import_graph(std::uint32_t n, std::uint32_t k, const std::uint32_t* ids,
                      const float* dists, const std::uint8_t* flags) {
    std::vector<std::vector<NeighborEntry>> rows(n, std::vector<NeighborEntry>(k));
    for (std::uint32_t u = 0; u < n; ++u)
        for (std::uint32_t i = 0; i < k; ++i) {
            const std::size_t p = std::size_t(u) * k + i;
            rows[u][i] = NeighborEntry{ids[p], dists[p], flags[p] != 0};
        }
    return KnnGraph::from_rows(k, rows);
}

void export_cands(const CandidateSet& c, std::uint32_t* cand_ids, std::uint32_t* new_counts,
                  std::uint32_t* old_counts) {
    const std::uint32_t n = c.n(), cap = c.cap();
    for (std::uint32_t u = 0; u < n; ++u) {
        const auto nw = c.new_ids(u);
        const auto od = c.old_ids(u);
        std::uint32_t* block = cand_ids + std::size_t(u) * 2 * cap;
        std::fill(block, block + 2 * cap, 0xffffffffu);
        std::copy(nw.begin(), nw.end(), block);
        std::copy(od.begin(), od.end(), block + cap);
        new_counts[u] = static_cast<std::uint32_t>(nw.size());
        old_counts[u] = static_cast<std::uint32_t>(od.size());
    }
}

CandidateSet import_cands(std::uint32_t n, std::uint32_t cap, const std::uint32_t* cand_ids,
                          const std::uint32_t* new_counts, const std::uint32_t* old_counts) {
    CandidateSet c(n, cap);
    std::vector<std::uint32_t> nc(new_counts, new_counts + n), oc(old_counts, old_counts + n);
    for (std::uint32_t u = 0; u < n; ++u) {
        const std::uint32_t* block = cand_ids + std::size_t(u) * 2 * cap;
        std::copy(block, block + nc[u], c.new_data(u));
        std::copy(block + cap, block + cap + oc[u], c.old_data(u));
    }
    c.set_counts(nc, oc);
    return c;
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// knng::run (descent.hpp:193-255). iter_* arrays need max_iterations+1 slots;
// *n_rows receives the metrics row count (iteration 0 = init). sigma (n, nullable)
// receives the reorder permutation when one was applied.
int ref_run(const float* data, std::uint32_t n, std::uint32_t d, std::uint32_t k,
            std::uint32_t cap, double delta, std::uint32_t max_iterations, int reorder,
            std::uint32_t reorder_after, std::uint64_t seed, std::uint32_t* out_ids,
            float* out_dists, std::uint8_t* out_flags, std::uint64_t* iter_evals,
            std::uint64_t* iter_changes, double* iter_wall, std::uint32_t* n_rows,
            double* total_wall, std::uint32_t* sigma) {
    return guarded([&] {
        const Dataset ds = make_dataset(data, n, d);
        RunParams p;
        p.k = k;
        p.max_candidates = cap;
        p.termination_delta = delta;
        p.max_iterations = max_iterations;
        p.reorder = reorder != 0;
        p.reorder_after_iteration = reorder_after;
        p.seed = seed;
        const RunResult r = run(ds, p);
        export_graph(r.graph, out_ids, out_dists, out_flags, nullptr);
        const auto& its = r.metrics.iterations;
        for (std::size_t i = 0; i < its.size(); ++i) {
            if (iter_evals) iter_evals[i] = its[i].dist_evals;
            if (iter_changes) iter_changes[i] = its[i].changes;
            if (iter_wall) iter_wall[i] = its[i].wall_time_s;
        }
        if (n_rows) *n_rows = static_cast<std::uint32_t>(its.size());
        if (total_wall) *total_wall = r.metrics.total_wall_time_s;
        if (sigma && r.permutation)
            std::copy(r.permutation->sigma.begin(), r.permutation->sigma.end(), sigma);
    });
}

// Replays run()'s loop (descent.hpp:201-228: same master Rng, same seeds, same
// calls, reorder off) up to iteration t and captures the fixed state of that
// iteration's local join: the heaps after select_turbo + flag_consumed, the
// candidate set, then the graph after the reference compute_step. t >= 1.
int ref_capture_step(const float* data, std::uint32_t n, std::uint32_t d, std::uint32_t k,
                     std::uint32_t cap, std::uint64_t seed, std::uint32_t t,
                     std::uint32_t* in_ids, float* in_dists, std::uint8_t* in_flags,
                     std::uint32_t* in_rev_deg, std::uint32_t* cand_ids,
                     std::uint32_t* new_counts, std::uint32_t* old_counts,
                     std::uint32_t* out_ids, float* out_dists, std::uint8_t* out_flags,
                     std::uint32_t* out_rev_deg, std::uint64_t* changes, std::uint64_t* evals) {
    return guarded([&] {
        if (t < 1) throw std::invalid_argument("ref_capture_step: t must be >= 1");
        const Dataset ds = make_dataset(data, n, d);
        EvalCounter counter;
        Rng master(seed);
        const std::uint64_t init_seed = master();
        KnnGraph g = KnnGraph::init_random(ds, k, init_seed, counter);
        CandidateSet cands(n, cap);
        for (std::uint32_t iter = 1; iter <= t; ++iter) {
            const std::uint64_t iter_seed = master();
            g.reset_change_count();
            select_turbo(g, iter_seed, cands);
            for (std::uint32_t u = 0; u < n; ++u) g.flag_consumed(u, cands.new_ids(u));
            if (iter == t) {
                export_graph(g, in_ids, in_dists, in_flags, in_rev_deg);
                export_cands(cands, cand_ids, new_counts, old_counts);
            }
            const std::uint64_t before = counter.dist_evals;
            const std::uint64_t c = compute_step(g, cands, ds, counter);
            if (iter == t) {
                export_graph(g, out_ids, out_dists, out_flags, out_rev_deg);
                if (changes) *changes = c;
                if (evals) *evals = counter.dist_evals - before;
            }
        }
    });
}

// compute_step (descent.hpp:82-153) on an injected state (graph via
// KnnGraph::from_rows, graph.hpp:70-93; candidates via CandidateSet).
int ref_compute_step(const float* data, std::uint32_t n, std::uint32_t d, std::uint32_t k,
                     std::uint32_t cap, const std::uint32_t* in_ids, const float* in_dists,
                     const std::uint8_t* in_flags, const std::uint32_t* cand_ids,
                     const std::uint32_t* new_counts, const std::uint32_t* old_counts,
                     int flat, std::uint32_t* out_ids, float* out_dists, std::uint8_t* out_flags,
                     std::uint32_t* out_rev_deg, std::uint64_t* changes, std::uint64_t* evals) {
    return guarded([&] {
        const Dataset ds = make_dataset(data, n, d);
        KnnGraph g = import_graph(n, k, in_ids, in_dists, in_flags);
        const CandidateSet c = import_cands(n, cap, cand_ids, new_counts, old_counts);
        EvalCounter counter;
        const std::uint64_t ch = flat ? compute_step_flat(g, c, ds, counter)
                                      : compute_step(g, c, ds, counter);
        export_graph(g, out_ids, out_dists, out_flags, out_rev_deg);
        if (changes) *changes = ch;
        if (evals) *evals = counter.dist_evals;
    });
}

// KnnGraph::init_random (graph.hpp:34-67).
int ref_init_random(const float* data, std::uint32_t n, std::uint32_t d, std::uint32_t k,
                    std::uint64_t seed, std::uint32_t* out_ids, float* out_dists,
                    std::uint8_t* out_flags, std::uint32_t* out_rev_deg, std::uint64_t* evals) {
    return guarded([&] {
        const Dataset ds = make_dataset(data, n, d);
        EvalCounter counter;
        const KnnGraph g = KnnGraph::init_random(ds, k, seed, counter);
        export_graph(g, out_ids, out_dists, out_flags, out_rev_deg);
        if (evals) *evals = counter.dist_evals;
    });
}

// select_turbo (selection.hpp:282-320) + flag_consumed (graph.hpp:133-143).
int ref_select_turbo(std::uint32_t n, std::uint32_t k, std::uint32_t cap,
                     const std::uint32_t* in_ids, const float* in_dists,
                     const std::uint8_t* in_flags, std::uint64_t seed, std::uint32_t* cand_ids,
                     std::uint32_t* new_counts, std::uint32_t* old_counts,
                     std::uint8_t* out_flags_after_consume) {
    return guarded([&] {
        KnnGraph g = import_graph(n, k, in_ids, in_dists, in_flags);
        CandidateSet c(n, cap);
        select_turbo(g, seed, c);
        export_cands(c, cand_ids, new_counts, old_counts);
        if (out_flags_after_consume) {
            for (std::uint32_t u = 0; u < n; ++u) g.flag_consumed(u, c.new_ids(u));
            // from_rows heapified the rows; report flags in the caller's entry order
            for (std::uint32_t u = 0; u < n; ++u)
                for (std::uint32_t i = 0; i < k; ++i) {
                    const std::uint32_t id = in_ids[std::size_t(u) * k + i];
                    for (std::uint32_t j = 0; j < k; ++j)
                        if (g.entry(u, j).id == id)
                            out_flags_after_consume[std::size_t(u) * k + i] =
                                g.entry(u, j).is_new ? 1 : 0;
                }
        }
    });
}

// brute_force_knng (oracle.hpp:92-127), unguarded.
int ref_brute_force(const float* data, std::uint32_t n, std::uint32_t d, std::uint32_t k,
                    std::uint32_t* out_ids, double* out_dists) {
    return guarded([&] {
        const Dataset ds = make_dataset(data, n, d);
        const ExactGraph ex = brute_force_knng(ds, k, true);
        std::copy(ex.ids.begin(), ex.ids.end(), out_ids);
        if (out_dists) std::copy(ex.dists.begin(), ex.dists.end(), out_dists);
    });
}

// recall (oracle.hpp:131-144) of a heap-order graph against exact ids.
int ref_recall(std::uint32_t n, std::uint32_t k, const std::uint32_t* approx_ids,
               const float* approx_dists, const std::uint32_t* exact_ids, double* out) {
    return guarded([&] {
        std::vector<std::uint8_t> flags(std::size_t(n) * k, 0);
        const KnnGraph g = import_graph(n, k, approx_ids, approx_dists, flags.data());
        ExactGraph ex;
        ex.k = k;
        ex.n = n;
        ex.ids.assign(exact_ids, exact_ids + std::size_t(n) * k);
        ex.dists.assign(std::size_t(n) * k, 0.0);
        *out = recall(g, ex);
    });
}

// greedy_cluster (reorder.hpp:22-50) on a graph given in heap order.
int ref_greedy_cluster(std::uint32_t n, std::uint32_t k, const std::uint32_t* ids,
                       const float* dists, const std::uint8_t* flags, std::uint32_t* sigma,
                       std::uint32_t* sigma_inv) {
    return guarded([&] {
        const KnnGraph g = import_graph(n, k, ids, dists, flags);
        const Permutation p = greedy_cluster(g);
        std::copy(p.sigma.begin(), p.sigma.end(), sigma);
        std::copy(p.sigma_inv.begin(), p.sigma_inv.end(), sigma_inv);
    });
}

// Distance kernels (distance.hpp:126-190). Rows are given as one contiguous
// m x d array; d must be the padded length the kernels run over.
float ref_l2_sq(const float* a, const float* b, std::uint32_t d) {
    EvalCounter c;
    return l2_sq(a, b, d, c);
}

int ref_block_l2_sq(const float* rows_a, std::uint32_t na, const float* rows_b,
                    std::uint32_t nb, std::uint32_t d, float* out) {
    return guarded([&] {
        std::vector<const float*> pa, pb;
        for (std::uint32_t i = 0; i < na; ++i) pa.push_back(rows_a + std::size_t(i) * d);
        for (std::uint32_t i = 0; i < nb; ++i) pb.push_back(rows_b + std::size_t(i) * d);
        EvalCounter c;
        block_l2_sq(std::span<const float* const>(pa), std::span<const float* const>(pb), d, out,
                    c);
    });
}

// Writes the m x m symmetric matrix (diagonal untouched) and the visit order
// (pairs i,j as 2*count u32) of mutual_block_distances.
int ref_mutual_block(const float* rows, std::uint32_t m, std::uint32_t d, float* out_matrix,
                     std::uint32_t* visit_pairs, std::uint64_t* n_visits) {
    return guarded([&] {
        std::vector<const float*> p;
        for (std::uint32_t i = 0; i < m; ++i) p.push_back(rows + std::size_t(i) * d);
        EvalCounter c;
        std::uint64_t count = 0;
        mutual_block_distances(std::span<const float* const>(p), d, c,
                               [&](std::uint32_t i, std::uint32_t j, float dist) {
                                   out_matrix[std::size_t(i) * m + j] = dist;
                                   out_matrix[std::size_t(j) * m + i] = dist;
                                   if (visit_pairs) {
                                       visit_pairs[2 * count] = i;
                                       visit_pairs[2 * count + 1] = j;
                                   }
                                   ++count;
                               });
        if (n_visits) *n_visits = count;
    });
}

// Reference generators (dataset.hpp:99-154); output unpadded n x d.
int ref_gen_gaussian(std::uint32_t n, std::uint32_t d, int single, std::uint64_t seed,
                     float* out) {
    return guarded([&] {
        const Dataset ds = gen_gaussian(n, d, single != 0, seed);
        for (std::uint32_t i = 0; i < n; ++i)
            std::memcpy(out + std::size_t(i) * d, ds.row(i), sizeof(float) * d);
    });
}

int ref_gen_clustered(std::uint32_t n, std::uint32_t d, std::uint32_t c, std::uint64_t seed,
                      float* out, std::uint32_t* labels) {
    return guarded([&] {
        const auto [ds, lab] = gen_clustered(n, d, c, seed);
        for (std::uint32_t i = 0; i < n; ++i)
            std::memcpy(out + std::size_t(i) * d, ds.row(i), sizeof(float) * d);
        std::copy(lab.labels.begin(), lab.labels.end(), labels);
    });
}

// Raw std::mt19937_64 stream (dataset.hpp:23) for pinning the restated engine.
void ref_mt64_stream(std::uint64_t seed, std::uint64_t* out, std::uint32_t count) {
    Rng r(seed);
    for (std::uint32_t i = 0; i < count; ++i) out[i] = r();
}

} // extern "C"
