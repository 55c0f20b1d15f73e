// knng_cuda_cli — the GPU path behind the reference CLI's own front end
// (SURVEY.md §8f rank 1-2).  Same subcommands, flags and file formats as
// `knng build` / `knng recall` (reference tools/knng_cli.cpp:129-153,207-222):
//
//   knng_cuda_cli build  --dataset D.knng --seed S [--k 20] [--max-candidates 50]
//                        [--max-iterations 30] [--delta 0.001] [--reorder]
//                        [--strategy turbo] [--compute blocked] [--device 0]
//                        [--graph-out G.csv] [--metrics-out M.csv]
//   knng_cuda_cli recall --graph G.csv --dataset D.knng [--k 20] [--device 0]
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
#include <map>
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

int cmd_build(const Args& a) {
    const Dataset data = load_dataset(a.need("--dataset"));
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
    const size_t nk = size_t(data.n) * p.k;
    std::vector<uint32_t> ids(nk);
    std::vector<float> dists(nk);
    std::vector<knng_cuda_iteration> its(p.max_iterations + 1);
    knng_cuda_metrics m;
    std::memset(&m, 0, sizeof m);
    m.iterations = its.data();
    m.capacity = uint32_t(its.size());
    check(knng_cuda_run(data.x.data(), data.n, data.d, &p, ids.data(), dists.data(), nullptr,
                        nullptr, &m));
    const std::string gout = a.get("--graph-out");
    if (!gout.empty()) {
        FILE* f = std::fopen(gout.c_str(), "w");
        if (!f) throw std::runtime_error("cannot open " + gout);
        std::fputs("node,neighbor,distance\n", f);
        // rows come back ascending by (distance, id): the export_csv order
        for (uint32_t u = 0; u < data.n; ++u)
            for (uint32_t i = 0; i < p.k; ++i)
                std::fprintf(f, "%u,%u,%.9g\n", u, ids[size_t(u) * p.k + i],
                             double(dists[size_t(u) * p.k + i]));
        if (std::fclose(f) != 0) throw std::runtime_error("write failed for " + gout);
    }
    const std::string mout = a.get("--metrics-out");
    if (!mout.empty()) {
        FILE* f = std::fopen(mout.c_str(), "w");
        if (!f) throw std::runtime_error("cannot open " + mout);
        std::fputs("iteration,wall_time_s,dist_evals,changes\n", f);
        for (uint32_t r = 0; r < std::min(m.n_rows, m.capacity); ++r)
            std::fprintf(f, "%u,%.6f,%llu,%llu\n", its[r].iteration, its[r].wall_time_s,
                         (unsigned long long)its[r].dist_evals,
                         (unsigned long long)its[r].changes);
        std::fprintf(f, "total,%.6f,%llu,%llu\n", m.total_wall_time_s,
                     (unsigned long long)m.total_dist_evals, (unsigned long long)m.total_changes);
        if (std::fclose(f) != 0) throw std::runtime_error("write failed for " + mout);
    }
    std::printf("n=%u d=%u iters=%u dist_evals=%llu total_s=%.3f\n", data.n, data.d,
                m.n_rows > 0 ? m.n_rows - 1 : 0, (unsigned long long)m.total_dist_evals,
                m.total_wall_time_s);
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
        if (argc < 2) throw std::runtime_error("usage: knng_cuda_cli build|recall [flags]");
        const std::string cmd = argv[1];
        if (cmd == "build") return cmd_build(parse(argc, argv, 2, {"--reorder"}));
        if (cmd == "recall") return cmd_recall(parse(argc, argv, 2, {}));
        throw std::runtime_error("unknown subcommand " + cmd + " (build | recall)");
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
