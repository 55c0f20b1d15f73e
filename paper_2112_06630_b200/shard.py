"""Multi-GPU NN-Descent: one process per GPU, vertex-range ownership.

Every rank keeps the whole dataset and a replica of the whole graph; it owns
the rows [rank * chunk, (rank + 1) * chunk).  Per iteration (reference loop
descent.hpp:219-243):

1. ``engine.step``: selection of the owned candidate lists over the replicated
   graph (per-edge Philox draws, so the lists do not depend on the sharding),
   local join of the owned active nodes, merges into owned rows, and records
   (target, id, distance) for targets owned elsewhere, grouped by owner;
2. ``all_to_all`` of the record counts, then of the records;
3. ``engine.merge`` of the received records into owned rows;
4. ``all_gather`` of the owned rows (keys, is_new flags, row maxima) into every
   replica, ``all_reduce`` of changes / evaluations / candidates, and the
   reference's termination test ``changes < delta * n * k``.

The collectives go through ``torch.distributed`` (NCCL over NVLink on GPUs; the
same runner drives a numpy engine over gloo in the CPU tests). The per-device
work is the CUDA library (:class:`GpuShardEngine`, C-ABI knng_cuda_shard_*).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N
from .knng import IterationMetrics, RunMetrics, RunParams, check


class _CudaArray:
    """Zero-copy view of a device pointer for torch.as_tensor."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape),
                                         "typestr": typestr, "strides": None, "version": 3}


def _device_view(ptr: int, count: int, typestr: str, device):
    import torch
    dtype = {"<i8": torch.int64, "<i4": torch.int32, "<f4": torch.float32}[typestr]
    if count == 0 or not ptr:
        return torch.empty(0, dtype=dtype, device=device)
    return torch.as_tensor(_CudaArray(ptr, (count,), typestr), device=device)


def seed_sequence(seed: int, count: int) -> np.ndarray:
    """std::mt19937_64(seed) outputs: [0] init seed, [i] iteration i
    (descent.hpp:201-221), from the library so every path agrees."""
    out = np.zeros(count, np.uint64)
    N.lib().knng_cuda_seed_sequence(seed & 0xFFFFFFFFFFFFFFFF, count, out)
    return out


class GpuShardEngine:
    """This rank's share of a sharded build on its GPU (knng_cuda_shard_*)."""

    def __init__(self, d_data, params: RunParams, rank: int, nranks: int):
        import torch
        self.torch = torch
        n, d = d_data.shape
        self.n, self.d, self.k = int(n), int(d), params.k
        self.rank, self.nranks = rank, nranks
        self.device = d_data.device
        self._data = d_data.contiguous()
        p = params._c()
        self._h = C.c_void_p()
        info = N.ShardInfo()
        check(N.lib().knng_cuda_shard_create(self._data.data_ptr(), self.n, self.d, C.byref(p),
                                             rank, nranks, None, C.byref(self._h),
                                             C.byref(info)))
        self.chunk, self.lo, self.hi = int(info.chunk), int(info.lo), int(info.hi)
        rows = int(info.rows_alloc)
        self.keys = _device_view(info.keys, rows * self.k, "<i8", self.device)
        self.flags = _device_view(info.flags, rows, "<i4", self.device)
        self.maxd = _device_view(info.maxd, rows, "<f4", self.device)

    def seeds(self, seed: int, count: int) -> np.ndarray:
        return seed_sequence(seed, count)

    def init(self, seed: int) -> None:
        check(N.lib().knng_cuda_shard_init(self._h, int(seed)))

    def step(self, seed: int):
        ctr = np.zeros(4, np.uint64)
        counts = np.zeros(self.nranks, np.uint64)
        ptr = C.c_void_p()
        check(N.lib().knng_cuda_shard_step(self._h, int(seed), ctr, counts, C.byref(ptr)))
        total = int(counts.sum())
        send = _device_view(ptr.value or 0, 3 * total, "<i4", self.device)
        return dict(evals=int(ctr[0]), cands=int(ctr[1]), active=int(ctr[3]),
                    send_counts=[int(c) for c in counts], send=send)

    def merge(self, recv) -> int:
        changes = np.zeros(1, np.uint64)
        recv = recv.contiguous()
        check(N.lib().knng_cuda_shard_merge(self._h, recv.data_ptr() if recv.numel() else None,
                                            recv.numel() // 3, changes))
        return int(changes[0])

    def sync(self) -> None:
        self.torch.cuda.current_stream(self.device).synchronize()

    def export(self):
        rows = self.hi - self.lo
        ids = self.torch.empty((rows, self.k), dtype=self.torch.int32, device=self.device)
        dists = self.torch.empty((rows, self.k), dtype=self.torch.float32, device=self.device)
        if rows:
            check(N.lib().knng_cuda_shard_export(self._h, ids.data_ptr(), dists.data_ptr()))
        return ids, dists

    def close(self) -> None:
        if self._h:
            N.lib().knng_cuda_shard_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class ShardedResult:
    ids: object              # (hi - lo, k) owned rows, sorted by (distance, id)
    dists: object
    lo: int
    hi: int
    metrics: RunMetrics = field(default_factory=RunMetrics)
    bytes_exchanged: int = 0  # records sent by this rank (all iterations)


def _allgather_rows(engine, group=None) -> None:
    import torch.distributed as dist
    r, P, chunk, k = engine.rank, engine.nranks, engine.chunk, engine.k
    for buf, width in ((engine.keys, k), (engine.flags, 1), (engine.maxd, 1)):
        parts = [buf[i * chunk * width:(i + 1) * chunk * width] for i in range(P)]
        dist.all_gather(parts, parts[r].clone(), group=group)


def run_sharded(engine, params: RunParams, group=None) -> ShardedResult:
    """The reference's run loop (descent.hpp:193-255) over P ranks."""
    import time

    import torch
    import torch.distributed as dist
    n, k, P = engine.n, engine.k, engine.nranks
    dev = engine.device
    seeds = engine.seeds(params.seed, params.max_iterations + 1)
    metrics = RunMetrics()
    t0 = time.perf_counter()
    engine.init(int(seeds[0]))
    _allgather_rows(engine, group)
    engine.sync()
    metrics.iterations.append(IterationMetrics(0, time.perf_counter() - t0, n * k, 0))
    threshold = params.termination_delta * n * k
    sent = 0
    for it in range(1, params.max_iterations + 1):
        t0 = time.perf_counter()
        st = engine.step(int(seeds[it]))
        send_counts = torch.tensor([3 * c for c in st["send_counts"]], dtype=torch.int64,
                                   device=dev)
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=group)
        rc = recv_counts.tolist()
        recv = torch.empty(int(sum(rc)), dtype=torch.int32, device=dev)
        dist.all_to_all_single(recv, st["send"], output_split_sizes=rc,
                               input_split_sizes=send_counts.tolist(), group=group)
        sent += 4 * int(sum(send_counts.tolist()))
        engine.sync()
        changes = engine.merge(recv)
        _allgather_rows(engine, group)
        tot = torch.tensor([changes, st["evals"], st["cands"]], dtype=torch.float64, device=dev)
        dist.all_reduce(tot, group=group)
        engine.sync()
        changes_all, evals_all, cands_all = (int(x) for x in tot.tolist())
        metrics.iterations.append(IterationMetrics(it, time.perf_counter() - t0, evals_all,
                                                   changes_all, cands_all))
        if changes_all < threshold:
            break
    for itm in metrics.iterations:
        metrics.total_wall_time_s += itm.wall_time_s
        metrics.total_dist_evals += itm.dist_evals
        metrics.total_changes += itm.changes
    ids, dists = engine.export()
    return ShardedResult(ids, dists, engine.lo, engine.hi, metrics, sent)


def gather_graph(res: ShardedResult, n: int, k: int, group=None):
    """All owned slices concatenated (every rank gets the full n x k graph)."""
    import torch
    import torch.distributed as dist
    P = dist.get_world_size(group)
    chunk = (n + P - 1) // P
    pad = chunk - (res.hi - res.lo)
    ids = torch.nn.functional.pad(res.ids, (0, 0, 0, pad)) if pad else res.ids
    dd = torch.nn.functional.pad(res.dists, (0, 0, 0, pad)) if pad else res.dists
    outs_i = [torch.empty_like(ids) for _ in range(P)]
    outs_d = [torch.empty_like(dd) for _ in range(P)]
    dist.all_gather(outs_i, ids.contiguous(), group=group)
    dist.all_gather(outs_d, dd.contiguous(), group=group)
    return torch.cat(outs_i)[:n], torch.cat(outs_d)[:n]
