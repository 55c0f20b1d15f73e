"""The multi-GPU protocol (paper_2112_06630_b200/shard.py: run_sharded) over
gloo on CPU with world_size 2: owned-range selection, local joins, the
record all-to-all, merges of received records and the row all-gathers must
give exactly the single-rank result (deterministic numpy shard engine)."""
import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_path, n, d, k, cap, iters, delta):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from paper_2112_06630_b200.knng import RunParams
    from paper_2112_06630_b200.shard import gather_graph, run_sharded
    from shard_ref_engine import NumpyShardEngine
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    data = np.random.default_rng(3).standard_normal((n, d)).astype(np.float32)
    eng = NumpyShardEngine(data, k, cap, rank, world)
    params = RunParams(k=k, max_candidates=cap, termination_delta=delta, max_iterations=iters,
                       seed=11)
    res = run_sharded(eng, params)
    ids, dists = gather_graph(res, n, k)
    if rank == 0:
        np.savez(out_path, ids=ids.numpy(), dists=dists.numpy(),
                 evals=np.array([it.dist_evals for it in res.metrics.iterations]),
                 changes=np.array([it.changes for it in res.metrics.iterations]))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, **kw):
    out = tempfile.mktemp(suffix=".npz")
    mp.spawn(_worker, args=(world, _free_port(), out, kw["n"], kw["d"], kw["k"], kw["cap"],
                            kw["iters"], kw["delta"]), nprocs=world, join=True)
    r = np.load(out)
    os.unlink(out)
    return r


CASE = dict(n=240, d=8, k=6, cap=10, iters=3, delta=1e-9)


@pytest.fixture(scope="module")
def single():
    return _run(1, **CASE)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_equals_single_rank(single, world):
    multi = _run(world, **CASE)
    assert np.array_equal(multi["ids"], single["ids"])
    assert np.array_equal(multi["dists"].view(np.uint32), single["dists"].view(np.uint32))
    # evaluations are a property of the lists, not of the sharding
    assert np.array_equal(multi["evals"], single["evals"])


def test_sharded_graph_improves(single):
    data = np.random.default_rng(3).standard_normal((CASE["n"], CASE["d"])).astype(np.float32)
    d2 = ((data[:, None, :].astype(np.float64) - data[None]) ** 2).sum(-1)
    np.fill_diagonal(d2, np.inf)
    exact = np.argsort(d2, axis=1)[:, : CASE["k"]]
    hits = sum(len(set(a) & set(b)) for a, b in zip(single["ids"].tolist(), exact.tolist()))
    assert hits / exact.size > 0.9
    # rows sorted, distances are the pairs' distances
    assert np.all(np.diff(single["dists"], axis=1) >= 0)
