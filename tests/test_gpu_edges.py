"""Edge cases of the GPU path: minimum and maximum sizes,
dimensions that are not multiples of 8, duplicate points (distance ties) and
degenerate all-equal data — each against the reference restatement where the
result is defined, or against the row invariants where any tie order is
valid."""
import numpy as np
import pytest

import paper_2112_06630_b200 as kg
from test_gpu_parity import compare_step

pytestmark = pytest.mark.gpu


def _rows_valid(ids, dists, n, k):
    assert ids.shape == (n, k)
    assert not np.any(ids == np.arange(n)[:, None])           # no self loops
    assert all(len(set(r)) == k for r in ids.tolist())        # distinct neighbours
    assert np.all(ids < n)
    assert np.all(np.diff(dists, axis=1) >= 0)                # sorted by distance


def test_minimum_n_gives_the_complete_graph(gpu):
    # n = k + 1: every node's k neighbours are all the other nodes
    for n, k, d in ((3, 2, 8), (9, 8, 5), (33, 32, 3)):
        data = np.random.default_rng(n).standard_normal((n, d), dtype=np.float32)
        res = kg.run(data, kg.RunParams(k=k, max_candidates=max(k, 2 * k)))
        _rows_valid(res.graph.ids, res.graph.dists, n, k)
        for u in range(n):
            assert sorted(res.graph.ids[u].tolist()) == [v for v in range(n) if v != u]


@pytest.mark.parametrize("n,d,k,cap,seed,t", [
    (1500, 16, 32, 64, 9, 1),   # the build's maximum k and max_candidates
    (1500, 16, 32, 64, 9, 2),
    (2000, 13, 12, 30, 3, 1),   # d % 8 != 0: zero-padded stride 16
    (2000, 5, 10, 20, 4, 2),    # d < 8: one partial 8-lane chunk
])
def test_step_parity_at_size_limits(gpu, restated, n, d, k, cap, seed, t):
    data = np.random.default_rng(seed).standard_normal((n, d), dtype=np.float32)
    gi, c, go, _, ev_ref = restated.capture_step(data, k, cap, seed, t)
    g, rev, ch, ev = kg.compute_step(data, gi.ids, gi.dists, gi.flags,
                                     kg.CandidateSet(c.ids, c.new_counts, c.old_counts))
    assert ev == ev_ref
    st = compare_step(gi, go, g, restated=restated, data=data)
    assert st["mismatch"] == 0 and st["flag_mismatch"] == 0, st
    assert st["bit_exact"] + st["other_path"] == st["common"], st


def test_max_sizes_recall_matches_reference(gpu, restated):
    n, d, k, cap = 3000, 16, 32, 64
    data = np.random.default_rng(17).standard_normal((n, d), dtype=np.float32)
    res = kg.run(data, kg.RunParams(k=k, max_candidates=cap, seed=2))
    ex, _ = kg.brute_force_knng(data, k)
    ref = restated.run(data, k=k, cap=cap, seed=2)
    assert kg.recall(res.graph.ids, ex) >= kg.recall(ref.graph.ids, ex) - 0.005


def test_duplicate_points_ties(gpu, restated):
    # 400 distinct points, each repeated 5 times: zero distances and exact ties
    base = np.random.default_rng(5).standard_normal((400, 24), dtype=np.float32)
    data = np.repeat(base, 5, axis=0)
    n, k = len(data), 10
    res = kg.run(data, kg.RunParams(k=k, max_candidates=30, seed=1))
    _rows_valid(res.graph.ids, res.graph.dists, n, k)
    # the 4 copies of a point are at distance 0 and must be found
    for u in range(0, n, 97):
        copies = {v for v in range(u - u % 5, u - u % 5 + 5) if v != u}
        assert copies <= set(res.graph.ids[u].tolist()), u
    ex, _ = kg.brute_force_knng(data, k)
    ref = restated.run(data, k=k, cap=30, seed=1)
    # recall against one exact answer of many (ties): both implementations alike
    assert abs(kg.recall(res.graph.ids, ex) - kg.recall(ref.graph.ids, ex)) < 0.05


def test_all_points_equal(gpu):
    data = np.ones((500, 8), np.float32)
    res = kg.run(data, kg.RunParams(k=6, max_candidates=12))
    _rows_valid(res.graph.ids, res.graph.dists, 500, 6)
    assert np.all(res.graph.dists == 0)


def test_iteration_observer(gpu):
    """The reference's IterationObserver (descent.hpp:184, called at :241):
    one call per iteration, in order, each with a sorted graph; without a
    reorder the last one is the returned graph."""
    import paper_2112_06630_b200 as kg
    data = np.random.default_rng(5).standard_normal((3000, 16)).astype(np.float32)
    seen = []

    def obs(it, g):
        assert np.all(np.diff(g.dists, axis=1) >= 0)
        seen.append((it, g.ids.copy(), g.dists.copy()))

    res = kg.run(data, kg.RunParams(k=10, max_candidates=20, seed=3), observer=obs)
    iters = len(res.metrics.iterations) - 1
    assert [s[0] for s in seen] == list(range(1, iters + 1))
    assert np.array_equal(seen[-1][1], res.graph.ids)
    assert np.array_equal(seen[-1][2].view(np.uint32), res.graph.dists.view(np.uint32))
    # with a reorder the observer sees the permuted labeling from that
    # iteration on; the returned graph is in original ids
    seen.clear()
    res2 = kg.run(data, kg.RunParams(k=10, max_candidates=20, seed=3, reorder=True,
                                     reorder_after_iteration=1), observer=obs)
    assert len(seen) == len(res2.metrics.iterations) - 1
    sig = res2.permutation
    assert np.array_equal(np.sort(seen[-1][1][sig], axis=1), np.sort(sig[res2.graph.ids], axis=1))


# zero-padded stride 104; stride == d with 77 MB of rows (more chunks than
# the 64 MiB ring has slots, so slots are reused)
@pytest.mark.parametrize("n,d", [(30000, 100), (200000, 96)])
def test_pinned_and_pageable_host_buffers_agree(gpu, n, d):
    """host_io.cu: pageable rows and results go through the pinned ring (above
    2 MiB), pinned ones are copied directly; both give the same graph as the
    device-resident entry point."""
    import torch
    k = 20
    data = np.random.default_rng(d).standard_normal((n, d), dtype=np.float32)
    p = kg.RunParams(k=k, max_candidates=30, seed=5, deterministic=True)
    a = kg.run(data, p)                                   # pageable in and out
    pinned = torch.empty((n, d), dtype=torch.float32, pin_memory=True)
    pinned.numpy()[:] = data
    b = kg.run(pinned.numpy(), p)                         # pinned in, pageable out
    assert a.metrics.h2d_bytes == b.metrics.h2d_bytes == data.nbytes
    np.testing.assert_array_equal(a.graph.ids, b.graph.ids)
    np.testing.assert_array_equal(a.graph.dists, b.graph.dists)
    np.testing.assert_array_equal(a.graph.flags, b.graph.flags)
    out = kg.KnnGraph(torch.empty((n, k), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32),
                      torch.empty((n, k), dtype=torch.float32, pin_memory=True).numpy(),
                      torch.empty((n, k), dtype=torch.uint8, pin_memory=True).numpy())
    c = kg.run(pinned.numpy(), p, out=out)                # pinned in and out (caller-owned)
    assert c.graph is out
    np.testing.assert_array_equal(a.graph.ids, out.ids)
    np.testing.assert_array_equal(a.graph.dists, out.dists)
    np.testing.assert_array_equal(a.graph.flags, out.flags)
    nof = kg.run(data, p, out=kg.KnnGraph(np.zeros((n, k), np.uint32), np.zeros((n, k), np.float32)))
    assert nof.graph.flags is None
    np.testing.assert_array_equal(a.graph.ids, nof.graph.ids)
    dev = torch.from_numpy(data).cuda()
    ids = torch.empty((n, k), dtype=torch.int32, device="cuda")
    dd = torch.empty((n, k), dtype=torch.float32, device="cuda")
    kg.run_device(dev.data_ptr(), n, d, p, ids.data_ptr(), dd.data_ptr())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(a.graph.ids, ids.cpu().numpy().view(np.uint32))
    np.testing.assert_array_equal(a.graph.dists, dd.cpu().numpy())
