// knng_cuda_cli — the GPU path behind the reference CLI's own front end
// (SURVEY.md §8f ranks 1, 2 and 4).  Same subcommands, flags and file formats
// as the reference's `knng` (tools/knng_cli.cpp:114-187, 193-269):
//
//   knng_cuda_cli generate --kind gaussian|gaussian-single|clustered --n N --d D
//                          [--c 8] --seed S --out D.knng [--labels-out L.csv]
//   knng_cuda_cli build  --dataset D.knng --seed S [--k 20] [--max-candidates 50]
//                        [--max-iterations 30] [--delta 0.001] [--reorder]
//                        [--strategy turbo] [--compute blocked] [--device 0]
//                        [--graph-out G.csv] [--metrics-out M.csv]
//   knng_cuda_cli recall --graph G.csv --dataset D.knng [--k 20] [--device 0]
//   knng_cuda_cli reorder-eval --dataset D.knng --labels L.csv --seed S --out W.csv
//                        [--k 20] [--window 2000] [--device 0]
//   knng_cuda_cli sweep  --kind K --n N1,N2,.. --d D1,.. [--c 8] --seed S --out M.csv
//                        [--k 20] [--max-candidates 50] [--reorder] [--device 0]
//
// `generate` draws from std::mt19937_64 with libstdc++'s normal distribution
// and std::shuffle, the generators the reference specifies
// (dataset.hpp:99-150), so the same seed gives the same points.
// `reorder-eval` runs one iteration with the locality reorder after it
// (knng_cli.cpp:223-241) and writes the window cluster fractions of the GPU
// permutation (reorder.hpp:61-86).  `sweep` writes the concatenated metrics
// rows of a build per grid point and, for a single d and >= 3 sizes, the
// least-squares slope of log(dist_evals) against log(n)
// (oracle.hpp:147-171, knng_cli.cpp:242-269).
//
// Formats (restated from their specifications, not copied):
//   dataset  KNNG binary v1, little-endian: "KNNG", u32 version 1, u64 n,
//            u64 d, n*d float32 row-major (dataset.hpp:188-233);
//   graph    CSV "node,neighbor,distance", rows of a node ascending by
//            (distance, id), distance printed with %.9g (graph.hpp:169-184);
//   metrics  CSV "iteration,wall_time_s,dist_evals,changes" plus a "total"
//            row (descent.hpp:53-67).
// `recall` computes the exact K-NNG with the GPU brute force
// (knng_cuda_bruteforce_knng, float64 distances, (dist, id) ties) instead of
// the reference's CPU one, so it has no 100k-point guard (oracle.hpp:46,96-97),
// and reports |approx ∩ exact| / (n k) (oracle.hpp:131-144).
//
// Errors print "error: <message>" and exit 1, like the reference's front end.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <cmath>
#include <map>
#include <numeric>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "knng_cuda.h"

namespace {

struct Dataset {
    uint32_t n = 0, d = 0;
    std::vector<float> x;  // n x d, unpadded
};

uint32_t get_u32(std::istream& is, const std::string& path, const char* what) {
    unsigned char b[4];
    if (!is.read(reinterpret_cast<char*>(b), 4))
        throw std::runtime_error(std::string("load_binary: ") + what + " in " + path);
    return uint32_t(b[0]) | uint32_t(b[1]) << 8 | uint32_t(b[2]) << 16 | uint32_t(b[3]) << 24;
}

uint64_t get_u64(std::istream& is, const std::string& path, const char* what) {
    const uint64_t lo = get_u32(is, path, what);
    return lo | uint64_t(get_u32(is, path, what)) << 32;
}

Dataset load_dataset(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw std::runtime_error("load_binary: cannot open " + path);
    char magic[4];
    if (!is.read(magic, 4) || std::memcmp(magic, "KNNG", 4) != 0)
        throw std::runtime_error("load_binary: bad magic in " + path);
    if (get_u32(is, path, "truncated header") != 1)
        throw std::runtime_error("load_binary: unsupported format version in " + path);
    const uint64_t n = get_u64(is, path, "truncated header");
    const uint64_t d = get_u64(is, path, "truncated header");
    if (n < 2 || d == 0 || n > 0xffffffffull || d > 0xffffffffull)
        throw std::runtime_error("load_binary: invalid dimensions in " + path);
    Dataset out;
    out.n = uint32_t(n);
    out.d = uint32_t(d);
    out.x.resize(size_t(n) * d);
    // little-endian IEEE-754 on every supported host: one bulk read
    if (!is.read(reinterpret_cast<char*>(out.x.data()), std::streamsize(sizeof(float) * out.x.size())))
        throw std::runtime_error("load_binary: truncated payload in " + path);
    return out;
}

struct Graph {
    uint32_t n = 0, k = 0;
    std::vector<uint32_t> ids;  // n x k
};

Graph read_graph_csv(const std::string& path) {
    std::ifstream is(path);
    if (!is) throw std::runtime_error("cannot open " + path);
    std::string line;
    if (!std::getline(is, line) || line != "node,neighbor,distance")
        throw std::runtime_error("bad graph header in " + path);
    std::vector<std::vector<uint32_t>> rows;
    while (std::getline(is, line)) {
        if (line.empty()) continue;
        unsigned node, nb;
        float dist;
        if (std::sscanf(line.c_str(), "%u,%u,%f", &node, &nb, &dist) != 3)
            throw std::runtime_error("bad graph row in " + path);
        if (node >= rows.size()) rows.resize(size_t(node) + 1);
        rows[node].push_back(nb);
    }
    if (rows.empty()) throw std::runtime_error("empty graph in " + path);
    Graph g;
    g.n = uint32_t(rows.size());
    g.k = uint32_t(rows[0].size());
    g.ids.resize(size_t(g.n) * g.k);
    for (uint32_t u = 0; u < g.n; ++u) {
        if (rows[u].size() != g.k) throw std::runtime_error("ragged graph rows in " + path);
        std::copy(rows[u].begin(), rows[u].end(), g.ids.begin() + size_t(u) * g.k);
    }
    return g;
}

void check(int rc) {
    if (rc != KNNG_CUDA_OK) throw std::runtime_error(knng_cuda_last_error());
}

struct Args {
    std::map<std::string, std::string> kv;
    std::vector<std::string> flags;
    bool has(const std::string& f) const {
        return kv.count(f) || std::find(flags.begin(), flags.end(), f) != flags.end();
    }
    std::string get(const std::string& f, const std::string& def = "") const {
        auto it = kv.find(f);
        return it == kv.end() ? def : it->second;
    }
    std::string need(const std::string& f) const {
        auto it = kv.find(f);
        if (it == kv.end()) throw std::runtime_error(f + " is required");
        return it->second;
    }
};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& bool_flags) {
    Args a;
    for (int i = first; i < argc; ++i) {
        const std::string f = argv[i];
        if (f.rfind("--", 0) != 0) throw std::runtime_error("unexpected argument " + f);
        if (std::find(bool_flags.begin(), bool_flags.end(), f) != bool_flags.end()) {
            a.flags.push_back(f);
        } else {
            if (i + 1 >= argc) throw std::runtime_error(f + " needs a value");
            a.kv[f] = argv[++i];
        }
    }
    return a;
}

uint64_t to_u64(const std::string& s, const std::string& f) {
    size_t pos = 0;
    const unsigned long long v = std::stoull(s, &pos);
    if (pos != s.size()) throw std::runtime_error("bad value for " + f + ": " + s);
    return v;
}

knng_cuda_params params_from(const Args& a) {
    knng_cuda_params p;
    knng_cuda_params_default(&p);
    p.seed = to_u64(a.need("--seed"), "--seed");
    p.k = uint32_t(to_u64(a.get("--k", "20"), "--k"));
    p.max_candidates = uint32_t(to_u64(a.get("--max-candidates", "50"), "--max-candidates"));
    p.max_iterations = uint32_t(to_u64(a.get("--max-iterations", "30"), "--max-iterations"));
    p.termination_delta = std::stod(a.get("--delta", "0.001"));
    p.reorder = a.has("--reorder") ? 1 : 0;
    p.device = int(to_u64(a.get("--device", "0"), "--device"));
    // the GPU path implements the reference defaults; naive / fused / flat
    // are its benchmark baselines (descent.hpp:24-27)
    if (a.get("--strategy", "turbo") != "turbo")
        throw std::runtime_error("--strategy: the GPU path implements turbo selection");
    if (a.get("--compute", "blocked") != "blocked")
        throw std::runtime_error("--compute: the GPU path implements the blocked join");
    return p;
}

struct BuildOut {
    std::vector<uint32_t> ids, sigma;
    std::vector<float> dists;
    std::vector<knng_cuda_iteration> its;
    knng_cuda_metrics m;
};

BuildOut build_graph(const Dataset& data, const knng_cuda_params& p, bool want_sigma = false) {
    BuildOut o;
    const size_t nk = size_t(data.n) * p.k;
    o.ids.resize(nk);
    o.dists.resize(nk);
    if (want_sigma) o.sigma.resize(data.n);
    o.its.resize(p.max_iterations + 1);
    std::memset(&o.m, 0, sizeof o.m);
    o.m.iterations = o.its.data();
    o.m.capacity = uint32_t(o.its.size());
    check(knng_cuda_run(data.x.data(), data.n, data.d, &p, o.ids.data(), o.dists.data(), nullptr,
                        want_sigma ? o.sigma.data() : nullptr, &o.m));
    return o;
}

void print_summary(const Dataset& data, const knng_cuda_metrics& m) {
    std::printf("n=%u d=%u iters=%u dist_evals=%llu total_s=%.3f\n", data.n, data.d,
                m.n_rows > 0 ? m.n_rows - 1 : 0, (unsigned long long)m.total_dist_evals,
                m.total_wall_time_s);
}

int cmd_build(const Args& a) {
    const Dataset data = load_dataset(a.need("--dataset"));
    const knng_cuda_params p = params_from(a);
    const BuildOut o = build_graph(data, p);
    const std::string gout = a.get("--graph-out");
    if (!gout.empty()) {
        FILE* f = std::fopen(gout.c_str(), "w");
        if (!f) throw std::runtime_error("cannot open " + gout);
        std::fputs("node,neighbor,distance\n", f);
        // rows come back ascending by (distance, id): the export_csv order
        for (uint32_t u = 0; u < data.n; ++u)
            for (uint32_t i = 0; i < p.k; ++i)
                std::fprintf(f, "%u,%u,%.9g\n", u, o.ids[size_t(u) * p.k + i],
                             double(o.dists[size_t(u) * p.k + i]));
        if (std::fclose(f) != 0) throw std::runtime_error("write failed for " + gout);
    }
    const std::string mout = a.get("--metrics-out");
    if (!mout.empty()) {
        FILE* f = std::fopen(mout.c_str(), "w");
        if (!f) throw std::runtime_error("cannot open " + mout);
        std::fputs("iteration,wall_time_s,dist_evals,changes\n", f);
        for (uint32_t r = 0; r < std::min(o.m.n_rows, o.m.capacity); ++r)
            std::fprintf(f, "%u,%.6f,%llu,%llu\n", o.its[r].iteration, o.its[r].wall_time_s,
                         (unsigned long long)o.its[r].dist_evals,
                         (unsigned long long)o.its[r].changes);
        std::fprintf(f, "total,%.6f,%llu,%llu\n", o.m.total_wall_time_s,
                     (unsigned long long)o.m.total_dist_evals, (unsigned long long)o.m.total_changes);
        if (std::fclose(f) != 0) throw std::runtime_error("write failed for " + mout);
    }
    print_summary(data, o.m);
    return 0;
}

// ---- generate (dataset.hpp:99-150): gaussian / gaussian-single / clustered
struct Generated {
    Dataset data;
    std::vector<uint32_t> labels;  // clustered only
};

Generated generate(const std::string& kind, uint32_t n, uint32_t d, uint32_t c, uint64_t seed) {
    if (n < 2 || d < 1) throw std::invalid_argument("generate: need n >= 2 and d >= 1");
    Generated g;
    g.data.n = n;
    g.data.d = d;
    g.data.x.assign(size_t(n) * d, 0.0f);
    std::mt19937_64 rng(seed);
    if (kind == "gaussian" || kind == "gaussian-single") {
        // N(0, 2) coordinates; the multi-cluster variant shifts coordinate
        // i mod d of point i by +1
        std::normal_distribution<float> gauss(0.0f, std::sqrt(2.0f));
        for (uint32_t i = 0; i < n; ++i) {
            float* r = g.data.x.data() + size_t(i) * d;
            for (uint32_t j = 0; j < d; ++j) r[j] = gauss(rng);
            if (kind == "gaussian") r[i % d] += 1.0f;
        }
        return g;
    }
    if (kind != "clustered") throw std::runtime_error("--kind: gaussian | gaussian-single | clustered");
    if (c < 2) throw std::invalid_argument("gen_clustered: need at least 2 clusters");
    if (n < 2 * c) throw std::invalid_argument("gen_clustered: need at least 2 points per cluster");
    // c unit-covariance Gaussians, n / c points each (the remainder to the
    // last), means on axis (cl mod d) at 10 sqrt(d) (1 + cl / d); then a
    // seeded shuffle of the point order
    std::normal_distribution<float> gauss(0.0f, 1.0f);
    const float scale = 10.0f * std::sqrt(float(d));
    std::vector<float> staged(size_t(n) * d);
    std::vector<uint32_t> lab(n);
    uint32_t at = 0;
    for (uint32_t cl = 0; cl < c; ++cl) {
        const uint32_t count = cl + 1 == c ? n - at : n / c;
        for (uint32_t i = 0; i < count; ++i, ++at) {
            float* r = staged.data() + size_t(at) * d;
            for (uint32_t j = 0; j < d; ++j) r[j] = gauss(rng);
            r[cl % d] += scale * float(1 + cl / d);
            lab[at] = cl;
        }
    }
    std::vector<uint32_t> order(n);
    std::iota(order.begin(), order.end(), 0u);
    std::shuffle(order.begin(), order.end(), rng);
    g.labels.resize(n);
    for (uint32_t i = 0; i < n; ++i) {
        std::copy_n(staged.data() + size_t(order[i]) * d, d, g.data.x.data() + size_t(i) * d);
        g.labels[i] = lab[order[i]];
    }
    return g;
}

void save_dataset(const Dataset& data, const std::string& path) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw std::runtime_error("cannot open " + path);
    auto put = [&](uint64_t v, int bytes) {
        for (int i = 0; i < bytes; ++i) os.put(char((v >> (8 * i)) & 0xff));
    };
    os.write("KNNG", 4);
    put(1, 4);
    put(data.n, 8);
    put(data.d, 8);
    os.write(reinterpret_cast<const char*>(data.x.data()),
             std::streamsize(sizeof(float) * data.x.size()));
    if (!os) throw std::runtime_error("write failed for " + path);
}

void write_labels(const std::vector<uint32_t>& labels, const std::string& path) {
    std::ofstream os(path);
    if (!os) throw std::runtime_error("cannot open " + path);
    os << "point,label\n";
    for (size_t i = 0; i < labels.size(); ++i) os << i << ',' << labels[i] << '\n';
    if (!os) throw std::runtime_error("write failed for " + path);
}

std::vector<uint32_t> read_labels(const std::string& path, uint32_t& clusters) {
    std::ifstream is(path);
    if (!is) throw std::runtime_error("cannot open " + path);
    std::string line;
    if (!std::getline(is, line) || line != "point,label")
        throw std::runtime_error("bad labels header in " + path);
    std::vector<uint32_t> out;
    clusters = 0;
    while (std::getline(is, line)) {
        if (line.empty()) continue;
        const size_t comma = line.find(',');
        if (comma == std::string::npos) throw std::runtime_error("bad labels row in " + path);
        const uint32_t v = uint32_t(std::stoul(line.substr(comma + 1)));
        out.push_back(v);
        clusters = std::max(clusters, v + 1);
    }
    return out;
}

std::vector<uint32_t> u32_list(const std::string& s, const std::string& f) {
    std::vector<uint32_t> out;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ','))
        if (!tok.empty()) out.push_back(uint32_t(to_u64(tok, f)));
    if (out.empty()) throw std::runtime_error(f + " needs at least one value");
    return out;
}

int cmd_generate(const Args& a) {
    const std::string kind = a.get("--kind", "gaussian");
    const Generated g = generate(kind, uint32_t(to_u64(a.need("--n"), "--n")),
                                 uint32_t(to_u64(a.need("--d"), "--d")),
                                 uint32_t(to_u64(a.get("--c", "8"), "--c")),
                                 to_u64(a.need("--seed"), "--seed"));
    const std::string out = a.need("--out");
    save_dataset(g.data, out);
    if (kind == "clustered") write_labels(g.labels, a.get("--labels-out", out + ".labels.csv"));
    return 0;
}

// window_cluster_fraction (reorder.hpp:61-86): windows of `window`
// consecutive permuted positions, starts advancing by window / 4, the last
// start n - window always included; the fraction of each cluster per window
int cmd_reorder_eval(const Args& a) {
    const Dataset data = load_dataset(a.need("--dataset"));
    uint32_t clusters = 0;
    const std::vector<uint32_t> labels = read_labels(a.need("--labels"), clusters);
    const uint32_t window = uint32_t(to_u64(a.get("--window", "2000"), "--window"));
    if (labels.size() != data.n)
        throw std::invalid_argument("window_cluster_fraction: labels/permutation size mismatch");
    if (window == 0 || data.n < window)
        throw std::invalid_argument("window_cluster_fraction: window larger than dataset");
    knng_cuda_params p;
    knng_cuda_params_default(&p);
    p.k = uint32_t(to_u64(a.get("--k", "20"), "--k"));
    p.seed = to_u64(a.need("--seed"), "--seed");
    p.device = int(to_u64(a.get("--device", "0"), "--device"));
    p.reorder = 1;
    p.reorder_after_iteration = 1;
    p.max_iterations = 1;
    const BuildOut o = build_graph(data, p, /*want_sigma=*/true);
    std::vector<uint32_t> inv(data.n);
    for (uint32_t i = 0; i < data.n; ++i) inv[o.sigma[i]] = i;
    const std::string out = a.need("--out");
    FILE* f = std::fopen(out.c_str(), "w");
    if (!f) throw std::runtime_error("cannot open " + out);
    std::fputs("window_start,cluster_id,fraction\n", f);
    const uint32_t step = std::max(1u, window / 4);
    std::vector<uint32_t> counts(clusters);
    for (uint32_t p0 = 0;;) {
        std::fill(counts.begin(), counts.end(), 0u);
        for (uint32_t q = p0; q < p0 + window; ++q) ++counts[labels[inv[q]]];
        for (uint32_t cl = 0; cl < clusters; ++cl)
            std::fprintf(f, "%u,%u,%.17g\n", p0, cl, double(counts[cl]) / window);
        if (p0 == data.n - window) break;
        p0 = std::min(p0 + step, data.n - window);
    }
    if (std::fclose(f) != 0) throw std::runtime_error("write failed for " + out);
    return 0;
}

// least-squares slope of log(evals) on log(n) (oracle.hpp:147-171)
double scaling_exponent(const std::vector<double>& n, const std::vector<double>& e) {
    if (n.size() != e.size() || n.size() < 3)
        throw std::invalid_argument("scaling_exponent: need at least 3 matched points");
    for (size_t i = 0; i < n.size(); ++i) {
        if (n[i] <= 0 || e[i] <= 0)
            throw std::invalid_argument("scaling_exponent: sizes and counts must be positive");
        if (i > 0 && n[i] <= n[i - 1])
            throw std::invalid_argument("scaling_exponent: sizes must be increasing");
    }
    double mx = 0, my = 0;
    for (size_t i = 0; i < n.size(); ++i) {
        mx += std::log(n[i]);
        my += std::log(e[i]);
    }
    mx /= double(n.size());
    my /= double(n.size());
    double sxy = 0, sxx = 0;
    for (size_t i = 0; i < n.size(); ++i) {
        const double dx = std::log(n[i]) - mx;
        sxy += dx * (std::log(e[i]) - my);
        sxx += dx * dx;
    }
    return sxy / sxx;
}

int cmd_sweep(const Args& a) {
    const std::string kind = a.get("--kind", "gaussian");
    const std::vector<uint32_t> ns = u32_list(a.need("--n"), "--n");
    const std::vector<uint32_t> ds = u32_list(a.need("--d"), "--d");
    const uint32_t c = uint32_t(to_u64(a.get("--c", "8"), "--c"));
    const knng_cuda_params p = params_from(a);
    const std::string out = a.need("--out");
    FILE* f = std::fopen(out.c_str(), "w");
    if (!f) throw std::runtime_error("cannot open " + out);
    std::fputs("n,d,iteration,wall_time_s,dist_evals,changes\n", f);
    std::vector<double> sizes, evals;
    for (uint32_t d : ds)
        for (uint32_t n : ns) {
            const Generated g = generate(kind, n, d, c, p.seed);
            const BuildOut o = build_graph(g.data, p);
            for (uint32_t r = 0; r < std::min(o.m.n_rows, o.m.capacity); ++r)
                std::fprintf(f, "%u,%u,%u,%.6f,%llu,%llu\n", n, d, o.its[r].iteration,
                             o.its[r].wall_time_s, (unsigned long long)o.its[r].dist_evals,
                             (unsigned long long)o.its[r].changes);
            std::fprintf(f, "%u,%u,total,%.6f,%llu,%llu\n", n, d, o.m.total_wall_time_s,
                         (unsigned long long)o.m.total_dist_evals,
                         (unsigned long long)o.m.total_changes);
            print_summary(g.data, o.m);
            sizes.push_back(n);
            evals.push_back(double(o.m.total_dist_evals));
        }
    if (std::fclose(f) != 0) throw std::runtime_error("write failed for " + out);
    if (ds.size() == 1 && sizes.size() >= 3)
        std::printf("scaling_exponent=%.4f\n", scaling_exponent(sizes, evals));
    return 0;
}

int cmd_recall(const Args& a) {
    const Dataset data = load_dataset(a.need("--dataset"));
    const Graph g = read_graph_csv(a.need("--graph"));
    const uint32_t k = uint32_t(to_u64(a.get("--k", "20"), "--k"));
    const int device = int(to_u64(a.get("--device", "0"), "--device"));
    if (g.k != k) throw std::runtime_error("graph k does not match --k");
    if (g.n != data.n) throw std::runtime_error("graph and dataset sizes differ");
    std::vector<uint32_t> ex(size_t(data.n) * k);
    std::vector<double> exd(ex.size());
    check(knng_cuda_bruteforce_knng(data.x.data(), data.n, data.d, k, ex.data(), exd.data(),
                                    device));
    uint64_t hit = 0;
    std::vector<uint32_t> a_row(k), e_row(k);
    for (uint32_t u = 0; u < data.n; ++u) {
        std::copy_n(g.ids.begin() + size_t(u) * k, k, a_row.begin());
        std::copy_n(ex.begin() + size_t(u) * k, k, e_row.begin());
        std::sort(a_row.begin(), a_row.end());
        std::sort(e_row.begin(), e_row.end());
        std::vector<uint32_t> both;
        std::set_intersection(a_row.begin(), a_row.end(), e_row.begin(), e_row.end(),
                              std::back_inserter(both));
        hit += both.size();
    }
    std::printf("recall=%.6f\n", double(hit) / (double(data.n) * k));
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 2)
            throw std::runtime_error(
                "usage: knng_cuda_cli generate|build|recall|reorder-eval|sweep [flags]");
        const std::string cmd = argv[1];
        if (cmd == "generate") return cmd_generate(parse(argc, argv, 2, {}));
        if (cmd == "build") return cmd_build(parse(argc, argv, 2, {"--reorder"}));
        if (cmd == "recall") return cmd_recall(parse(argc, argv, 2, {}));
        if (cmd == "reorder-eval") return cmd_reorder_eval(parse(argc, argv, 2, {}));
        if (cmd == "sweep") return cmd_sweep(parse(argc, argv, 2, {"--reorder"}));
        throw std::runtime_error("unknown subcommand " + cmd +
                                 " (generate | build | recall | reorder-eval | sweep)");
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
