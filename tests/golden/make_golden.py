"""Writes the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

    PYTHONPATH=. python tests/golden/make_golden.py

Every output below comes from oracle/_ref/libknng_ref.so, i.e. the unmodified
reference headers (/root/reference/proj/include/knng) compiled by
oracle/Makefile — never from this repo's own code.  Inputs are small seeded
numpy arrays stored next to the outputs, so the fixtures are self-contained
and the tests that read them need neither /root/reference nor a rebuild.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def main() -> None:
    if not oracle.available("reference"):
        oracle.build("reference")
    R = oracle.load("reference")
    rng = np.random.default_rng(20261020)
    out = {}

    # distance kernels: every tile shape at the reference test dims
    # (test_distance.cpp:98-121, acceptance.cpp:74-129)
    for d in (8, 24, 256, 784, 960):
        A = rng.standard_normal((5, d), dtype=np.float32)
        B = rng.standard_normal((5, d), dtype=np.float32)
        out[f"kern_a_{d}"] = A
        out[f"kern_b_{d}"] = B
        for na in range(1, 6):
            for nb in range(1, 6):
                out[f"kern_block_{d}_{na}x{nb}"] = R.block_l2_sq(A[:na], B[:nb])
        M = rng.standard_normal((13, d), dtype=np.float32)
        out[f"kern_mut_rows_{d}"] = M
        mat, visits = R.mutual_block(M)
        out[f"kern_mut_{d}"] = mat
        out[f"kern_mut_visits_{d}"] = visits
        out[f"kern_scalar_{d}"] = np.array([R.l2_sq(A[0], B[0])], np.float32)

    # std::mt19937_64 stream
    out["mt64_seed5"] = R.mt64_stream(5, 2048)

    # whole runs (knng::run): heap-order graph and per-iteration metrics
    runs = {
        "run_u8": (rng.random((1500, 8), dtype=np.float32), dict(k=10, cap=10, seed=5)),
        "run_g24": (rng.standard_normal((800, 24), dtype=np.float32), dict(k=8, cap=15, seed=7)),
        "run_g24_reorder": (None, dict(k=8, cap=15, seed=7, reorder=True)),
    }
    for name, (data, kw) in runs.items():
        if data is None:
            data = out["run_g24_data"]
        out[f"{name}_data"] = data
        r = R.run(data, **kw)
        out[f"{name}_ids"] = r.graph.ids
        out[f"{name}_dists"] = r.graph.dists
        out[f"{name}_flags"] = r.graph.flags
        out[f"{name}_evals"] = r.iter_evals
        out[f"{name}_changes"] = r.iter_changes
        if r.sigma is not None:
            out[f"{name}_sigma"] = r.sigma

    # single join step from a fixed state (capture after select + flag_consumed)
    data = rng.standard_normal((600, 24), dtype=np.float32)
    out["step_data"] = data
    for t in (1, 2, 4):
        gi, c, go, ch, ev = R.capture_step(data, 8, 15, 11, t)
        for key, arr in (("in_ids", gi.ids), ("in_dists", gi.dists), ("in_flags", gi.flags),
                         ("in_rev", gi.rev_deg), ("cand", c.ids), ("nc", c.new_counts),
                         ("oc", c.old_counts), ("out_ids", go.ids), ("out_dists", go.dists),
                         ("out_flags", go.flags), ("out_rev", go.rev_deg)):
            out[f"step{t}_{key}"] = arr
        out[f"step{t}_changes"] = np.array([ch], np.uint64)
        out[f"step{t}_evals"] = np.array([ev], np.uint64)

    # init_random and select_turbo on their own
    data = rng.random((300, 8), dtype=np.float32)
    out["init_data"] = data
    g, ev = R.init_random(data, 6, 99)
    out["init_ids"], out["init_dists"], out["init_flags"], out["init_rev"] = (
        g.ids, g.dists, g.flags, g.rev_deg)
    c, fa = R.select_turbo(g, 10, 500)
    out["sel_cand"], out["sel_nc"], out["sel_oc"], out["sel_flags_after"] = (
        c.ids, c.new_counts, c.old_counts, fa)

    # brute force (double, (dist,id) order)
    data = rng.standard_normal((400, 16), dtype=np.float32)
    data[7] = data[3]  # a duplicate point: mutual neighbours at distance 0
    out["bf_data"] = data
    out["bf_ids"], out["bf_dists"] = R.brute_force(data, 7)

    np.savez_compressed(os.path.join(HERE, "reference_fixtures.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_fixtures.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
