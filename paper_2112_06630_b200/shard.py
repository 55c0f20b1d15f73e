"""Multi-GPU NN-Descent: one process per GPU, vertex-range ownership.

Every rank keeps the whole dataset; it owns the rows [rank * chunk,
(rank + 1) * chunk): their graph rows, candidate lists, joins and merges.
Only the row maxima (n floats, the join prefilter's bound) are replicated.
Per iteration (reference loop descent.hpp:219-243):

1. ``engine.degree``: partial in-degree of the owned rows' edges,
   ``all_reduce`` (sum) -> the global in-degree (turbo's deg = k + in-degree);
2. ``engine.sample``: sampling over the owned rows' edges only; reverse offers
   for rows owned elsewhere (accepted here) are grouped by owner,
   ``all_to_all`` -> ``engine.offers`` inserts the received ones;
3. ``engine.step``: finalize, local join of the owned active nodes, merges
   into owned rows, and pre-reduced records (target, id, distance) for rows
   owned elsewhere (<= k per target), ``all_to_all`` -> ``engine.merge``;
4. ``all_gather`` of the owned row maxima, ``all_reduce`` of changes /
   evaluations / candidates, and the reference's termination test
   ``changes < delta * n * k``.

Per-edge Philox draws keyed by the global edge index make the sampled lists
independent of the sharding.  The collectives go through
``torch.distributed`` (NCCL over NVLink on GPUs; the same runner drives a
numpy engine over gloo in the CPU tests) on the library's stream (the shard
is created on torch's current stream), so no host synchronisation orders
them; the host reads only the counts each variable-size exchange needs and
the iteration's counters.  One process driving N GPUs:
``paper_2112_06630_b200.run_multi`` (C-ABI knng_cuda_run_multi, peer copies).
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

    def __init__(self, d_data, params: RunParams, rank: int, nranks: int, stream=None):
        import torch
        self.torch = torch
        n, d = d_data.shape
        self.n, self.d, self.k = int(n), int(d), params.k
        self.rank, self.nranks = rank, nranks
        self.device = d_data.device
        self._data = d_data.contiguous()
        if stream is None:  # torch's current stream: the collectives order after our kernels
            stream = torch.cuda.current_stream(self.device).cuda_stream
            if stream == 0:
                stream = 1  # cudaStreamLegacy: the default stream itself, not a library stream
        p = params._c()
        self._h = C.c_void_p()
        info = N.ShardInfo()
        check(N.lib().knng_cuda_shard_create(self._data.data_ptr(), self.n, self.d, C.byref(p),
                                             rank, nranks, stream or None, C.byref(self._h),
                                             C.byref(info)))
        self._views(info)
        self.sigma = self.sigma_inv = None

    def _views(self, info) -> None:
        self.chunk, self.lo, self.hi = int(info.chunk), int(info.lo), int(info.hi)
        self.seg_cap = int(info.seg_cap)
        rows = int(info.rows_alloc)
        self.keys = _device_view(info.keys, rows * self.k, "<i8", self.device)
        self.flags = _device_view(info.flags, rows, "<i4", self.device)
        self.maxd = _device_view(info.maxd, rows, "<f4", self.device)
        self.indeg = _device_view(info.indeg, self.n, "<i4", self.device)

    def reorder(self):
        """The locality reorder (descent.hpp:230-235) once every shard's rows
        have been all-gathered into keys / flags / maxd: sigma (the same on
        every shard), data and graph permuted; (sigma, sigma_inv) as int32
        device views for the final remap."""
        info = N.ShardInfo()
        ps, pi = C.c_void_p(), C.c_void_p()
        check(N.lib().knng_cuda_shard_reorder(self._h, C.byref(info), C.byref(ps), C.byref(pi)))
        self._views(info)
        self.sigma = _device_view(ps.value, self.n, "<i4", self.device)
        self.sigma_inv = _device_view(pi.value, self.n, "<i4", self.device)
        return self.sigma, self.sigma_inv

    def seeds(self, seed: int, count: int) -> np.ndarray:
        return seed_sequence(seed, count)

    def init(self, seed: int) -> None:
        check(N.lib().knng_cuda_shard_init(self._h, int(seed)))

    def degree(self):
        """Partial in-degree of the owned rows' edges (int32 view, in place)."""
        check(N.lib().knng_cuda_shard_degree(self._h))
        return self.indeg

    def sample(self, seed: int):
        """(send_counts, segments): accepted reverse offers per owner rank, as
        int32 views of 4 words per record."""
        counts = np.zeros(self.nranks, np.uint64)
        ptr = C.c_void_p()
        check(N.lib().knng_cuda_shard_sample(self._h, int(seed), counts, C.byref(ptr)))
        allrec = _device_view(ptr.value or 0, 4 * self.seg_cap * self.nranks, "<i4", self.device)
        segs = [allrec[4 * r * self.seg_cap: 4 * (r * self.seg_cap + int(c))]
                for r, c in enumerate(counts)]
        return [int(c) for c in counts], segs

    def offers(self, recv) -> None:
        recv = recv.contiguous()
        check(N.lib().knng_cuda_shard_offers(self._h, recv.data_ptr() if recv.numel() else None,
                                             recv.numel() // 4))

    def step(self):
        ctr = np.zeros(4, np.uint64)
        counts = np.zeros(self.nranks, np.uint64)
        ptr = C.c_void_p()
        check(N.lib().knng_cuda_shard_step(self._h, ctr, counts, C.byref(ptr)))
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

    def metrics(self, capacity: int = 256) -> RunMetrics:
        """This shard's share: per-kernel times and one row per iteration
        (evaluations, candidates, inserts into owned rows, join-kernel ms)."""
        from .knng import _metrics
        m, rows = _metrics(capacity)
        check(N.lib().knng_cuda_shard_metrics(self._h, C.byref(m)))
        return RunMetrics._from_c(m, rows)

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
    sigma: object = None      # after a reorder: rows / ids above are in sigma's order


def _staged(t, group=None) -> bool:
    """Device tensors over a host-only backend (gloo) go through host memory;
    NCCL takes them in place."""
    import torch.distributed as dist
    return t.device.type == "cuda" and dist.get_backend(group) == "gloo"


def _all_reduce(t, group=None) -> None:
    import torch.distributed as dist
    if _staged(t, group):
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, group=group)


def _all_to_all_single(out, inp, out_splits=None, in_splits=None, group=None) -> None:
    import torch.distributed as dist
    if _staged(out, group):
        h = out.new_empty(out.shape, device="cpu")
        dist.all_to_all_single(h, inp.cpu(), output_split_sizes=out_splits,
                               input_split_sizes=in_splits, group=group)
        out.copy_(h)
    else:
        dist.all_to_all_single(out, inp, output_split_sizes=out_splits,
                               input_split_sizes=in_splits, group=group)


def _all_gather(parts, mine, group=None) -> None:
    import torch.distributed as dist
    if _staged(mine, group):
        hp = [p.new_empty(p.shape, device="cpu") for p in parts]
        dist.all_gather(hp, mine.cpu(), group=group)
        for p, h in zip(parts, hp):
            p.copy_(h)
    else:
        dist.all_gather(parts, mine, group=group)


def _exchange(segs: List, counts: List[int], width: int, dtype, dev, group=None):
    """Variable-size all-to-all of per-destination segments (width words per
    record); returns the concatenated received records."""
    import torch
    import torch.distributed as dist
    P = len(counts)
    send_counts = torch.tensor(counts, dtype=torch.int64, device=dev)
    recv_counts = torch.empty_like(send_counts)
    _all_to_all_single(recv_counts, send_counts, group=group)
    rc = recv_counts.tolist()  # the one host read this exchange needs
    parts = [segs[r] for r in range(P) if counts[r]]
    send = torch.cat(parts) if parts else torch.empty(0, dtype=dtype, device=dev)
    recv = torch.empty(width * int(sum(rc)), dtype=dtype, device=dev)
    _all_to_all_single(recv, send, [width * int(c) for c in rc],
                       [width * int(c) for c in counts], group=group)
    return recv


def _allgather_rows(engine, group=None) -> None:
    """Every shard's owned rows (keys, flags, row maxima) into every shard."""
    r, P, chunk, k = engine.rank, engine.nranks, engine.chunk, engine.k
    for buf, width in ((engine.keys, k), (engine.flags, 1), (engine.maxd, 1)):
        parts = [buf[i * chunk * width:(i + 1) * chunk * width] for i in range(P)]
        _all_gather(parts, parts[r].clone(), group=group)


def _allgather_maxd(engine, group=None) -> None:
    import torch.distributed as dist
    r, P, chunk = engine.rank, engine.nranks, engine.chunk
    parts = [engine.maxd[i * chunk:(i + 1) * chunk] for i in range(P)]
    _all_gather(parts, parts[r].clone(), group=group)


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
    _allgather_maxd(engine, group)
    engine.sync()
    metrics.iterations.append(IterationMetrics(0, time.perf_counter() - t0, n * k, 0))
    threshold = params.termination_delta * n * k
    sent = 0
    for it in range(1, params.max_iterations + 1):
        t0 = time.perf_counter()
        _all_reduce(engine.degree(), group=group)
        counts, segs = engine.sample(int(seeds[it]))
        recv = _exchange([s for s in segs], counts, 4, torch.int32, dev, group)
        engine.offers(recv)
        sent += 16 * sum(counts)
        st = engine.step()
        sc = st["send_counts"]
        offs = np.concatenate([[0], np.cumsum(sc)]).astype(np.int64)
        rsegs = [st["send"][3 * offs[r]: 3 * offs[r + 1]] for r in range(P)]
        recv = _exchange(rsegs, sc, 3, torch.int32, dev, group)
        sent += 12 * sum(sc)
        changes = engine.merge(recv)
        _allgather_maxd(engine, group)
        tot = torch.tensor([changes, st["evals"], st["cands"]], dtype=torch.float64, device=dev)
        _all_reduce(tot, group=group)
        changes_all, evals_all, cands_all = (int(x) for x in tot.tolist())
        # the locality reorder (descent.hpp:230-235): every shard gathers the
        # whole graph and computes the same sigma; the shards then own
        # contiguous ranges of sigma
        if (params.reorder and getattr(engine, "sigma", None) is None
                and it == params.reorder_after_iteration and hasattr(engine, "reorder")):
            _allgather_rows(engine, group)
            engine.reorder()
        metrics.iterations.append(IterationMetrics(it, time.perf_counter() - t0, evals_all,
                                                   changes_all, cands_all))
        if changes_all < threshold:
            break
    engine.sync()
    for itm in metrics.iterations:
        metrics.total_wall_time_s += itm.wall_time_s
        metrics.total_dist_evals += itm.dist_evals
        metrics.total_changes += itm.changes
    ids, dists = engine.export()
    return ShardedResult(ids, dists, engine.lo, engine.hi, metrics, sent,
                         getattr(engine, "sigma", None))


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
    _all_gather(outs_i, ids.contiguous(), group=group)
    _all_gather(outs_d, dd.contiguous(), group=group)
    ids_all, d_all = torch.cat(outs_i)[:n], torch.cat(outs_d)[:n]
    if res.sigma is not None:
        # back to the caller's ids (descent.hpp:245): row u is permuted row
        # sigma[u], ids renamed by sigma_inv, rows re-sorted by (distance, id)
        sigma = res.sigma.long()
        inv = torch.empty_like(sigma)
        inv[sigma] = torch.arange(n, device=sigma.device)
        ids_all = inv[ids_all[sigma].long()]
        d_all = d_all[sigma]
        key = (d_all.contiguous().view(torch.int32).long() << 32) | ids_all
        order = torch.argsort(key, dim=1)
        ids_all = torch.gather(ids_all, 1, order).int()
        d_all = torch.gather(d_all, 1, order)
    return ids_all, d_all
