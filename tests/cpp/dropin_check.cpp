// Drop-in check: the reference's own caller code, with knng::run swapped for
// knng::cuda::run (proj/include/knng/cuda.hpp), against the reference's own
// brute force and recall (oracle.hpp).  Built only where the reference headers
// exist (tests/cpp/Makefile); prints one line "dropin <status> ...".
#include <cstdio>
#include <exception>
#include <stdexcept>

#include "knng/cuda.hpp"
#include "knng/knng.hpp"

int main() {
    using namespace knng;
    // parameter errors keep the reference's exception type (test_descent.cpp:12-27)
    try {
        const Dataset data = gen_gaussian(30, 8, true, 1);
        RunParams bad;
        bad.k = 1;
        cuda::run(data, bad);
        std::printf("dropin FAIL invalid_argument not raised\n");
        return 1;
    } catch (const std::invalid_argument&) {
    }
    const Dataset data = gen_gaussian(4000, 8, false, 7);
    RunParams params;
    params.k = 20;
    params.seed = 13;
    try {
        // the reference's IterationObserver (descent.hpp:184,241): one call per
        // iteration, in order, with the graph as it stands after it
        std::uint32_t calls = 0, last_it = 0;
        double last_recall = -1.0;
        const ExactGraph exact = brute_force_knng(data, 20);
        const RunResult gpu = cuda::run(data, params, [&](std::uint32_t it, const KnnGraph& g) {
            ++calls;
            last_it = it;
            last_recall = recall(g, exact);
        });
        const RunResult cpu = run(data, params);
        const double rg = recall(gpu.graph, exact), rc = recall(cpu.graph, exact);
        const bool obs_ok = calls == gpu.metrics.iterations.size() - 1 &&
                            last_it == calls && last_recall == rg;
        const bool ok = rg >= rc - 0.005 && obs_ok;
        std::printf("dropin %s recall gpu %.4f cpu %.4f iterations gpu %zu cpu %zu observer "
                    "calls %u last recall %.4f\n",
                    ok ? "OK" : "FAIL", rg, rc, gpu.metrics.iterations.size() - 1,
                    cpu.metrics.iterations.size() - 1, calls, last_recall);
        return ok ? 0 : 1;
    } catch (const std::runtime_error& e) {
        std::printf("dropin NODEVICE %s\n", e.what());
        return 3;
    }
}
