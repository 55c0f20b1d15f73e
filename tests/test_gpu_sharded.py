"""The sharded (multi-GPU) path on one GPU: world_size 1 over NCCL exercises the
CUDA shard engine (knng_cuda_shard_*) end to end, including the record
export / all-to-all / merge machinery with an empty exchange, and must match
the single-GPU build's quality.  (More ranks than GPUs is not run: ranks whose
kernels wait on each other must not share a device — B200_PROFILING.md.)"""
import os
import socket

import numpy as np
import pytest

import paper_2112_06630_b200 as kg
from paper_2112_06630_b200 import datasets

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_world():
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_sharded_world1_matches_single_gpu(gpu, nccl_world):
    import torch
    from paper_2112_06630_b200.shard import GpuShardEngine, gather_graph, run_sharded
    cfg = datasets.CONFIGS["C1"]
    data = datasets.generate(cfg)
    params = kg.RunParams(k=cfg.k, max_candidates=cfg.cap, seed=0)
    eng = GpuShardEngine(torch.from_numpy(data).cuda(), params, 0, 1)
    res = run_sharded(eng, params)
    ids, dists = gather_graph(res, cfg.n, cfg.k)
    ids = ids.cpu().numpy().astype(np.uint32)
    ex, _ = kg.brute_force_knng(data, cfg.k)
    single = kg.run(data, params)
    r_sh = kg.recall(ids, ex)
    r_single = kg.recall(single.graph.ids, ex)
    assert r_sh >= r_single - 0.005, (r_sh, r_single)
    # same seeds, same per-edge draws: the same number of iterations +-1
    assert abs(len(res.metrics.iterations) - len(single.metrics.iterations)) <= 1
    assert res.metrics.iterations[0].dist_evals == cfg.n * cfg.k
    d = dists.cpu().numpy()
    assert np.all(np.diff(d, axis=1) >= 0)
    eng.close()


def test_shard_step_exports_nothing_with_one_rank(gpu, nccl_world):
    import torch
    from paper_2112_06630_b200.shard import GpuShardEngine
    data = np.random.default_rng(0).standard_normal((2000, 24)).astype(np.float32)
    params = kg.RunParams(k=8, max_candidates=16, seed=3)
    eng = GpuShardEngine(torch.from_numpy(data).cuda(), params, 0, 1)
    eng.init(1)
    indeg = eng.degree()
    torch.cuda.synchronize()
    assert int(indeg.sum()) == 2000 * 8  # one rank owns every edge
    counts, segs = eng.sample(2)
    assert counts == [0] and segs[0].numel() == 0  # no reverse offers leave the rank
    eng.offers(torch.empty(0, dtype=torch.int32, device="cuda"))
    st = eng.step()
    assert st["send_counts"] == [0] and st["send"].numel() == 0
    assert st["evals"] > 0 and st["active"] > 0
    assert eng.merge(torch.empty(0, dtype=torch.int32, device="cuda")) >= 0
    eng.close()


def _two_rank_build(data, params, k):
    """Two shard engines of a 2-rank split in ONE process, sequential kernels
    on one stream (nothing waits on another rank); the exchanges are done here
    by hand.  Returns (graph ids, per-iteration record checks)."""
    import torch
    from paper_2112_06630_b200.shard import GpuShardEngine, seed_sequence
    n = data.shape[0]
    dd = torch.from_numpy(data).cuda()
    engs = [GpuShardEngine(dd, params, r, 2) for r in range(2)]
    seeds = seed_sequence(params.seed, 31)
    chunk = engs[0].chunk

    def allgather_maxd():
        for r in range(2):
            src = engs[r].maxd[r * chunk:(r + 1) * chunk]
            engs[1 - r].maxd[r * chunk:(r + 1) * chunk].copy_(src)

    for e in engs:
        e.init(int(seeds[0]))
    allgather_maxd()
    for it in range(1, 31):
        parts = [e.degree().clone() for e in engs]
        total = parts[0] + parts[1]
        assert int(total.sum()) == n * k  # every edge counted once
        for e in engs:
            e.indeg.copy_(total)
        samples = [e.sample(int(seeds[it])) for e in engs]
        for r in range(2):
            counts, segs = samples[r]
            assert counts[r] == 0  # local offers never leave the rank
            recs = segs[1 - r].view(-1, 4)
            if recs.numel():
                tv = recs[:, 0].cpu().numpy()
                other = engs[1 - r]
                assert np.all((tv >= other.lo) & (tv < other.hi))
        for r in range(2):
            engs[r].offers(samples[1 - r][1][r].clone())
        steps = [e.step() for e in engs]
        changes = 0
        for r in range(2):
            c = steps[r]["send_counts"]
            assert c[r] == 0  # nothing addressed to itself
            recs = steps[r]["send"].view(-1, 3)
            t = recs[:, 0].cpu().numpy()
            other = 1 - r
            assert np.all((t >= engs[other].lo) & (t < engs[other].hi))
            # pre-reduced export: at most k records per remote target
            if len(t):
                assert np.bincount(t).max() <= k
        for r in range(2):
            changes += engs[r].merge(steps[1 - r]["send"].clone())
        allgather_maxd()
        if changes < params.termination_delta * n * k:
            break
    ids = torch.cat([e.export()[0] for e in engs]).cpu().numpy().astype(np.uint32)
    for e in engs:
        e.close()
    return ids


@pytest.mark.parametrize("kind,shard_u8", [
    ("C1", "1"),
    # C2-shaped data has hub targets; the FP32 join on the shards and the
    # byte-valued one, after earlier engines left non-zero pool memory behind
    ("C2", "0"),
    ("C2", "1"),
    ("C4", "1"),
])
def test_shard_engine_two_ranks_one_process_exchange(gpu, monkeypatch, kind, shard_u8):
    """A 2-rank split through the C-ABI phases (degree, sample, offers, step,
    merge) with the exchanges done by hand: offers and records go only to the
    owner, records are pre-reduced, and the graph's recall matches the
    single-GPU build."""
    monkeypatch.setenv("KNNG_SHARD_U8", shard_u8)
    cfg = datasets.CONFIGS[kind]
    data = datasets.generate(cfg, n=12000) if kind == "C4" else datasets.generate(cfg)[:12000]
    k = cfg.k
    params = kg.RunParams(k=k, max_candidates=cfg.cap, seed=0)
    ids = _two_rank_build(data, params, k)
    ex, _ = kg.brute_force_knng(data, k)
    single = kg.run(data, params)
    r_sh, r_single = kg.recall(ids, ex), kg.recall(single.graph.ids, ex)
    assert abs(r_sh - r_single) <= 0.005, (r_sh, r_single)


@pytest.mark.parametrize("kind,n,shards", [
    ("C1", None, 2),
    ("C1", None, 3),
    ("C2", 12000, 2),
    ("C3", 20000, 4),
    ("C4", 20000, 2),
    ("C4", 20000, 8),
])
def test_run_multi_matches_single_gpu(gpu, kind, n, shards):
    """knng_cuda_run_multi: the vertex-sharded build driven from one process
    (peer copies between the shards' streams; on one GPU every shard shares
    the device).  Recall within 0.5 pp of the single-GPU build from the same
    seed, the initial graph's evaluations counted once, rows sorted."""
    cfg = datasets.CONFIGS[kind]
    if n is None:
        data = datasets.generate(cfg)
    elif kind in ("C3", "C4"):
        data = datasets.generate(cfg, n=n)
    else:
        data = datasets.generate(cfg)[:n]
    params = kg.RunParams(k=cfg.k, max_candidates=cfg.cap, seed=0)
    ids, dists, m = kg.run_multi(data, params, num_gpus=shards)
    single = kg.run(data, params)
    ex, _ = kg.brute_force_knng(data, cfg.k)
    r_multi, r_single = kg.recall(ids, ex), kg.recall(single.graph.ids, ex)
    assert abs(r_multi - r_single) <= 0.005, (r_multi, r_single)
    assert m.iterations[0].dist_evals == data.shape[0] * cfg.k
    assert abs(len(m.iterations) - len(single.metrics.iterations)) <= 2
    assert np.all(np.diff(dists, axis=1) >= 0)
    assert all(len(set(r)) == cfg.k for r in ids.tolist())
    assert not np.any(ids == np.arange(data.shape[0])[:, None])
    # the distances are the pairs' true distances (to FP32 rounding)
    i = np.arange(0, data.shape[0], 97)
    d64 = ((data[i, None, :].astype(np.float64) - data[ids[i]].astype(np.float64)) ** 2).sum(-1)
    assert np.allclose(dists[i], d64, rtol=1e-4, atol=1e-4)


def test_nndescent_l2_num_gpus(gpu):
    """The north-star entry point with num_gpus > 1 runs the sharded build."""
    cfg = datasets.CONFIGS["C1"]
    data = datasets.generate(cfg)
    ids, dists, m = kg.nndescent_l2(data, k=20, sample_rate=1.0, seed=0, num_gpus=2)
    ex, _ = kg.brute_force_knng(data, 20)
    single = kg.run(data, kg.RunParams(k=20, max_candidates=20, seed=0))
    assert abs(kg.recall(ids, ex) - kg.recall(single.graph.ids, ex)) <= 0.005


@pytest.mark.parametrize("kind,n,shards", [("C1", None, 2), ("C4", 20000, 4), ("C3", 20000, 3)])
def test_run_multi_reorder(gpu, kind, n, shards):
    """The locality reorder on shards (descent.hpp:230-235, 245): sigma from
    the whole graph, every shard's data and graph permuted, the shards then
    owning contiguous ranges of sigma; the returned graph is in the caller's
    ids.  Recall within 0.01 of the build without reorder
    (test_descent.cpp:211-224) and within 0.5 pp of the single-GPU reordered
    build."""
    cfg = datasets.CONFIGS[kind]
    data = datasets.generate(cfg) if n is None else datasets.generate(cfg, n=n)
    base = kg.RunParams(k=cfg.k, max_candidates=cfg.cap, seed=0)
    reo = kg.RunParams(k=cfg.k, max_candidates=cfg.cap, seed=0, reorder=True,
                       reorder_after_iteration=1)
    ids, dists, m = kg.run_multi(data, reo, num_gpus=shards)
    ex, _ = kg.brute_force_knng(data, cfg.k)
    r_multi = kg.recall(ids, ex)
    r_plain = kg.recall(kg.run(data, base).graph.ids, ex)
    r_single_reo = kg.recall(kg.run(data, reo).graph.ids, ex)
    assert r_multi >= r_plain - 0.01, (r_multi, r_plain)
    assert abs(r_multi - r_single_reo) <= 0.005, (r_multi, r_single_reo)
    assert np.all(np.diff(dists, axis=1) >= 0)
    assert not np.any(ids == np.arange(data.shape[0])[:, None])
    i = np.arange(0, data.shape[0], 101)
    d64 = ((data[i, None, :].astype(np.float64) - data[ids[i]].astype(np.float64)) ** 2).sum(-1)
    assert np.allclose(dists[i], d64, rtol=1e-4, atol=1e-4)


def _mp_worker(rank, world, port, out_path, kind, n, reorder=False):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_2112_06630_b200 as kg2
    from paper_2112_06630_b200 import datasets as ds
    from paper_2112_06630_b200.shard import GpuShardEngine, gather_graph, run_sharded
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    cfg = ds.CONFIGS[kind]
    data = ds.generate(cfg, n=n) if kind in ("C3", "C4") else ds.generate(cfg)[:n]
    params = kg2.RunParams(k=cfg.k, max_candidates=cfg.cap, seed=0, reorder=reorder,
                           reorder_after_iteration=1)
    eng = GpuShardEngine(torch.from_numpy(data).cuda(), params, rank, world)
    res = run_sharded(eng, params)
    ids, dists = gather_graph(res, data.shape[0], cfg.k)
    if rank == 0:
        np.savez(out_path, ids=ids.cpu().numpy().astype(np.uint32), dists=dists.cpu().numpy(),
                 iters=len(res.metrics.iterations) - 1,
                 evals=np.array([it.dist_evals for it in res.metrics.iterations]))
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("kind,n,world,reorder", [("C1", 10000, 2, False),
                                                  ("C4", 20000, 3, False),
                                                  ("C2", 12000, 2, False),
                                                  ("C4", 20000, 2, True),
                                                  ("C1", 10000, 3, True)])
def test_run_sharded_multiprocess(gpu, kind, n, world, reorder):
    """shard.py's run_sharded in separate processes (the torchrun path of
    bench.py --gpus N), each rank a real CUDA shard engine; the GPU is shared,
    so the collectives go over gloo through host memory (NCCL does not
    allow two ranks on one GPU).  Recall within 0.5 pp of the single-GPU
    build; the initial graph's evaluations counted once."""
    import tempfile

    import torch.multiprocessing as mp
    out = tempfile.mktemp(suffix=".npz")
    mp.spawn(_mp_worker, args=(world, _port(), out, kind, n, reorder), nprocs=world, join=True)
    r = np.load(out)
    os.unlink(out)
    cfg = datasets.CONFIGS[kind]
    data = datasets.generate(cfg, n=n) if kind in ("C3", "C4") else datasets.generate(cfg)[:n]
    params = kg.RunParams(k=cfg.k, max_candidates=cfg.cap, seed=0)
    single = kg.run(data, params)
    ex, _ = kg.brute_force_knng(data, cfg.k)
    r_mp, r_single = kg.recall(r["ids"], ex), kg.recall(single.graph.ids, ex)
    # with the reorder (shards own sigma ranges): within 0.01 of the plain
    # build (test_descent.cpp:211-224)
    assert abs(r_mp - r_single) <= (0.01 if reorder else 0.005), (r_mp, r_single)
    assert int(r["evals"][0]) == n * cfg.k
    assert not np.any(r["ids"] == np.arange(n)[:, None])
    i = np.arange(0, n, 97)
    d64 = ((data[i, None, :].astype(np.float64) - data[r["ids"][i]].astype(np.float64)) ** 2).sum(-1)
    assert np.allclose(r["dists"][i], d64, rtol=1e-4, atol=1e-4)
    assert np.all(np.diff(r["dists"], axis=1) >= 0)


@pytest.mark.parametrize("n,k,shards", [(12, 3, 8), (50, 5, 8), (200, 10, 7)])
def test_run_multi_tiny_and_empty_shards(gpu, n, k, shards):
    """More shards than rows per shard, some owning no rows at all: the
    exchanges with empty segments and the termination still work, and on a
    tiny set the build reaches the exact K-NNG like the single-GPU one."""
    data = np.random.default_rng(n).standard_normal((n, 6)).astype(np.float32)
    params = kg.RunParams(k=k, max_candidates=2 * k, seed=1)
    ids, dists, m = kg.run_multi(data, params, num_gpus=shards)
    ex, _ = kg.brute_force_knng(data, k)
    single = kg.run(data, params)
    assert kg.recall(ids, ex) >= kg.recall(single.graph.ids, ex) - 0.02
    assert all(len(set(r)) == k for r in ids.tolist())
    assert not np.any(ids == np.arange(n)[:, None])
    assert np.all(np.diff(dists, axis=1) >= 0)
