"""Host-side mirror of the reference's knng interface over libknng_cuda.so.

Same names, argument meaning and error behaviour as the reference's
proj/include/knng headers (cited per function), so callers and tests read
like the reference's own.  Every computation runs in the CUDA library; this
module only validates, marshals and wraps results.
"""
from __future__ import annotations

import ctypes as C
import io
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N
from ._native import InvalidArgument, KnngCudaError, check

__all__ = [
    "RunParams", "IterationMetrics", "RunMetrics", "KnnGraph", "RunResult", "CandidateSet",
    "run", "run_device", "nndescent_l2", "compute_step", "candidate_distances", "init_random",
    "select_turbo", "brute_force_knng", "recall", "locality_permutation", "flop_count",
    "InvalidArgument", "KnngCudaError", "device_count",
]


def device_count() -> int:
    return int(N.lib().knng_cuda_device_count())


def flop_count(dist_evals: int, d: int) -> int:
    """flop_count (distance.hpp:19-21): evals * (3d - 1)."""
    return int(dist_evals) * (3 * int(d) - 1)


@dataclass
class RunParams:
    """knng::RunParams (descent.hpp:18-36); strategy turbo, blocked join."""
    k: int = 20
    max_candidates: int = 50
    termination_delta: float = 0.001
    max_iterations: int = 30
    reorder: bool = False
    reorder_after_iteration: int = 1
    seed: int = 0
    device: int = 0
    profile: bool = False
    # seed-deterministic build: the same graph for the same seed
    # (acceptance.cpp:383-408); DESIGN.md §4
    deterministic: bool = False

    def validate(self) -> None:
        """RunParams::validate (descent.hpp:29-35)."""
        if self.k < 2:
            raise InvalidArgument("RunParams: k must be at least 2")
        if self.max_candidates < self.k:
            raise InvalidArgument("RunParams: max_candidates must be at least k")
        if not (0.0 < self.termination_delta < 1.0):
            raise InvalidArgument("RunParams: termination_delta must be in (0,1)")

    def _c(self) -> N.Params:
        p = N.Params()
        p.k = self.k
        p.max_candidates = self.max_candidates
        p.termination_delta = self.termination_delta
        p.max_iterations = self.max_iterations
        p.reorder = int(self.reorder)
        p.reorder_after_iteration = self.reorder_after_iteration
        p.seed = self.seed & 0xFFFFFFFFFFFFFFFF
        p.device = self.device
        p.profile = int(self.profile)
        p.deterministic = int(self.deterministic)
        return p


@dataclass
class IterationMetrics:
    """knng::IterationMetrics (descent.hpp:38-43)."""
    iteration: int
    wall_time_s: float
    dist_evals: int
    changes: int
    join_candidates: int = 0
    join_ms: float = 0.0


@dataclass
class RunMetrics:
    """knng::RunMetrics (descent.hpp:45-68) plus device-side accounting."""
    iterations: List[IterationMetrics] = field(default_factory=list)
    total_wall_time_s: float = 0.0
    total_dist_evals: int = 0
    total_changes: int = 0
    final_recall: Optional[float] = None
    kernel_ms: dict = field(default_factory=dict)
    kernel_launches: dict = field(default_factory=dict)
    join_candidates: int = 0
    join_evals: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0

    def write_csv(self, os: io.TextIOBase) -> None:
        """`iteration,wall_time_s,dist_evals,changes` + totals (descent.hpp:53-67)."""
        os.write("iteration,wall_time_s,dist_evals,changes\n")
        for it in self.iterations:
            os.write(f"{it.iteration},{it.wall_time_s:.6f},{it.dist_evals},{it.changes}\n")
        os.write(f"total,{self.total_wall_time_s:.6f},{self.total_dist_evals},"
                 f"{self.total_changes}\n")

    @staticmethod
    def _from_c(m: N.Metrics, rows) -> "RunMetrics":
        out = RunMetrics()
        for i in range(min(m.n_rows, m.capacity)):
            r = rows[i]
            out.iterations.append(IterationMetrics(int(r.iteration), float(r.wall_time_s),
                                                   int(r.dist_evals), int(r.changes),
                                                   int(r.join_candidates), float(r.join_ms)))
        out.total_wall_time_s = float(m.total_wall_time_s)
        out.total_dist_evals = int(m.total_dist_evals)
        out.total_changes = int(m.total_changes)
        out.kernel_ms = {n: float(m.kernel_ms[i]) for i, n in enumerate(N.KERNEL_NAMES)}
        out.kernel_launches = {n: int(m.kernel_launches[i]) for i, n in enumerate(N.KERNEL_NAMES)}
        out.join_candidates = int(m.join_candidates)
        out.join_evals = int(m.join_evals)
        out.h2d_bytes = int(m.h2d_bytes)
        out.d2h_bytes = int(m.d2h_bytes)
        return out


def _metrics(capacity: int):
    rows = (N.Iteration * max(1, capacity))()
    m = N.Metrics()
    m.iterations = C.cast(rows, C.POINTER(N.Iteration))
    m.capacity = capacity
    return m, rows


@dataclass
class KnnGraph:
    """The K-NN graph as returned: rows sorted by (distance, id)."""
    ids: np.ndarray                 # (n, k) uint32
    dists: np.ndarray               # (n, k) float32 squared L2
    flags: Optional[np.ndarray] = None  # (n, k) uint8, 1 = is_new

    @property
    def n(self) -> int:
        return int(self.ids.shape[0])

    @property
    def k(self) -> int:
        return int(self.ids.shape[1])

    def row(self, u: int):
        return list(zip(self.ids[u].tolist(), self.dists[u].tolist()))

    def max_dist(self, u: int) -> float:
        return float(self.dists[u].max())

    def reverse_degree(self) -> np.ndarray:
        """k + in-degree per node (KnnGraph::reverse_degree, graph.hpp:98)."""
        return (self.k + np.bincount(self.ids.ravel(), minlength=self.n)).astype(np.uint32)

    def export_csv(self, os: io.TextIOBase) -> None:
        """KnnGraph::export_csv (graph.hpp:169-184): rows by (distance, id)."""
        os.write("node,neighbor,distance\n")
        for u in range(self.n):
            order = np.lexsort((self.ids[u], self.dists[u]))
            for i in order:
                os.write(f"{u},{int(self.ids[u, i])},{float(self.dists[u, i]):.9g}\n")


@dataclass
class RunResult:
    """knng::RunResult (descent.hpp:70-74)."""
    graph: KnnGraph
    metrics: RunMetrics
    permutation: Optional[np.ndarray] = None  # sigma (n,) when reordered


@dataclass
class CandidateSet:
    """CandidateSet (selection.hpp:22-89): per node new list then old list."""
    ids: np.ndarray          # (n, 2*cap) uint32
    new_counts: np.ndarray   # (n,) uint32
    old_counts: np.ndarray   # (n,) uint32

    @property
    def cap(self) -> int:
        return int(self.ids.shape[1] // 2)

    def new_ids(self, u: int) -> np.ndarray:
        return self.ids[u, : self.new_counts[u]]

    def old_ids(self, u: int) -> np.ndarray:
        return self.ids[u, self.cap: self.cap + self.old_counts[u]]


def _as_data(data) -> np.ndarray:
    data = np.ascontiguousarray(data, dtype=np.float32)
    if data.ndim != 2:
        raise InvalidArgument("data must be an n x d array")
    return data


def _out_array(a, name, shape, dtype):
    if (not isinstance(a, np.ndarray) or a.shape != shape or a.dtype != dtype
            or not a.flags.c_contiguous or not a.flags.writeable):
        raise InvalidArgument(f"out.{name} must be a writeable C-contiguous {np.dtype(dtype).name} "
                              f"array of shape {shape}")
    return a


def run(data, params: RunParams = RunParams(), observer=None,
        out: Optional[KnnGraph] = None) -> RunResult:
    """knng::run (descent.hpp:193-255) on the GPU; host arrays in and out.

    observer(iteration, KnnGraph): the reference's IterationObserver
    (descent.hpp:184, called at :241), after each iteration in the run's
    current labeling (permuted ids after a reorder).

    out: caller-owned result arrays (n x k uint32 ids, float32 dists, uint8
    flags or None), e.g. page-locked ones reused across builds; the returned
    graph is `out`.  Without it the result goes to fresh arrays."""
    data = _as_data(data)
    params.validate()
    n, d = data.shape
    if n <= params.k:
        raise InvalidArgument("run: need n > k")
    k = params.k
    if out is None:
        ids = np.zeros((n, k), np.uint32)
        dists = np.zeros((n, k), np.float32)
        flags = np.zeros((n, k), np.uint8)
    else:
        ids = _out_array(out.ids, "ids", (n, k), np.uint32)
        dists = _out_array(out.dists, "dists", (n, k), np.float32)
        flags = None if out.flags is None else _out_array(out.flags, "flags", (n, k), np.uint8)
    sigma = np.zeros(n, np.uint32) if params.reorder else None
    m, rows = _metrics(params.max_iterations + 1)
    p = params._c()
    cb = None
    if observer is not None:
        def _obs(it, nn, kk, pi, pd, pf, _user):
            cnt = nn * kk
            g = KnnGraph(np.ctypeslib.as_array(pi, (cnt,)).reshape(nn, kk).copy(),
                         np.ctypeslib.as_array(pd, (cnt,)).reshape(nn, kk).copy(),
                         np.ctypeslib.as_array(pf, (cnt,)).reshape(nn, kk).copy())
            observer(int(it), g)
        cb = N.OBSERVER(_obs)
        p.observer = C.cast(cb, C.c_void_p)
    check(N.lib().knng_cuda_run(data.ctypes.data, n, d, C.byref(p), ids.ctypes.data,
                                dists.ctypes.data, flags.ctypes.data if flags is not None else None,
                                sigma.ctypes.data if sigma is not None else None, C.byref(m)))
    del cb
    return RunResult(out if out is not None else KnnGraph(ids, dists, flags),
                     RunMetrics._from_c(m, rows), sigma)


def run_multi(data, params: RunParams = RunParams(), num_gpus: int = 2, devices=None):
    """knng::run over num_gpus vertex shards in this process (C-ABI
    knng_cuda_run_multi; shard r on devices[r], default r % device count).
    Returns (ids, dists, metrics)."""
    data = _as_data(data)
    params.validate()
    n, d = data.shape
    if n <= params.k:
        raise InvalidArgument("run: need n > k")
    k = params.k
    ids = np.zeros((n, k), np.uint32)
    dists = np.zeros((n, k), np.float32)
    m, rows = _metrics(params.max_iterations + 1)
    p = params._c()
    dev = None
    if devices is not None:
        dev = (C.c_int * num_gpus)(*devices)
    check(N.lib().knng_cuda_run_multi(data, n, d, C.byref(p), num_gpus, dev, ids, dists,
                                      C.byref(m)))
    return ids, dists, RunMetrics._from_c(m, rows)


def run_device(data_ptr: int, n: int, d: int, params: RunParams, out_ids_ptr: int,
               out_dists_ptr: int, stream: int = 0) -> RunMetrics:
    """knng::run on device-resident buffers (raw device pointers, e.g.
    torch.Tensor.data_ptr()); outputs n x k ids / squared distances."""
    params.validate()
    m, rows = _metrics(params.max_iterations + 1)
    p = params._c()
    check(N.lib().knng_cuda_run_device(data_ptr, n, d, C.byref(p), out_ids_ptr, out_dists_ptr,
                                       C.byref(m), stream or None))
    return RunMetrics._from_c(m, rows)


def nndescent_l2(data, k: int, sample_rate: float, delta: float = 0.001, seed: int = 0,
                 max_iterations: int = 30, num_gpus: int = 1):
    """The north-star entry: (ids, dists, metrics); max_candidates = lround(rho*k)."""
    data = _as_data(data)
    n, d = data.shape
    ids = np.zeros((n, k), np.uint32)
    dists = np.zeros((n, k), np.float32)
    m, rows = _metrics(max_iterations + 1)
    check(N.lib().knng_cuda_nndescent_l2(data, n, d, k, sample_rate, delta, seed,
                                         max_iterations, num_gpus, ids, dists, C.byref(m)))
    return ids, dists, RunMetrics._from_c(m, rows)


def compute_step(data, ids, dists, flags, cands: CandidateSet, device: int = 0):
    """compute_step (descent.hpp:82-153) from a fixed state.

    Returns (KnnGraph with sorted rows, reverse_degree, changes, evals)."""
    data = _as_data(data)
    n, d = data.shape
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    k = ids.shape[1]
    o_ids = np.zeros((n, k), np.uint32)
    o_d = np.zeros((n, k), np.float32)
    o_f = np.zeros((n, k), np.uint8)
    rev = np.zeros(n, np.uint32)
    ch = np.zeros(1, np.uint64)
    ev = np.zeros(1, np.uint64)
    check(N.lib().knng_cuda_local_join(
        data, n, d, k, cands.cap, ids, np.ascontiguousarray(dists, dtype=np.float32),
        np.ascontiguousarray(flags, dtype=np.uint8), np.ascontiguousarray(cands.ids, np.uint32),
        np.ascontiguousarray(cands.new_counts, np.uint32),
        np.ascontiguousarray(cands.old_counts, np.uint32), o_ids, o_d, o_f, rev, ch, ev, device))
    return KnnGraph(o_ids, o_d, o_f), rev, int(ch[0]), int(ev[0])


def candidate_distances(data, cands: CandidateSet, device: int = 0):
    """The join's distance stage: {u: D_u} with D_u of shape (nn, nn + no);
    entries of the new x new block with j <= i are NaN."""
    data = _as_data(data)
    n, d = data.shape
    nc = np.ascontiguousarray(cands.new_counts, np.uint32)
    oc = np.ascontiguousarray(cands.old_counts, np.uint32)
    sizes = nc.astype(np.uint64) * (nc.astype(np.uint64) + oc.astype(np.uint64))
    offsets = np.zeros(n, np.uint64)
    if n > 1:
        offsets[1:] = np.cumsum(sizes)[:-1]
    total = int(sizes.sum())
    out = np.full(max(1, total), np.nan, np.float32)
    check(N.lib().knng_cuda_candidate_distances(data, n, d, cands.cap,
                                                np.ascontiguousarray(cands.ids, np.uint32), nc,
                                                oc, offsets, out, total, device))
    res = {}
    for u in np.nonzero(nc)[0]:
        a, b = int(nc[u]), int(nc[u] + oc[u])
        res[int(u)] = out[int(offsets[u]): int(offsets[u]) + a * b].reshape(a, b)
    return res


def init_random(data, k: int, seed: int, device: int = 0):
    """KnnGraph::init_random (graph.hpp:34-67): (graph, reverse_degree, evals)."""
    data = _as_data(data)
    n, d = data.shape
    ids = np.zeros((n, k), np.uint32)
    dists = np.zeros((n, k), np.float32)
    flags = np.zeros((n, k), np.uint8)
    rev = np.zeros(n, np.uint32)
    ev = np.zeros(1, np.uint64)
    check(N.lib().knng_cuda_init_random(data, n, d, k, seed, ids, dists, flags, rev, ev, device))
    return KnnGraph(ids, dists, flags), rev, int(ev[0])


def select_turbo(ids, dists, flags, cap: int, seed: int, device: int = 0):
    """select_turbo + flag_consumed (selection.hpp:282-320, graph.hpp:133-143).

    Returns (CandidateSet, flags after consumption in the input entry order)."""
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    n, k = ids.shape
    cids = np.zeros((n, 2 * cap), np.uint32)
    nc = np.zeros(n, np.uint32)
    oc = np.zeros(n, np.uint32)
    fa = np.zeros((n, k), np.uint8)
    check(N.lib().knng_cuda_select(n, k, cap, ids, np.ascontiguousarray(dists, np.float32),
                                   np.ascontiguousarray(flags, np.uint8), seed, cids, nc, oc, fa,
                                   device))
    return CandidateSet(cids, nc, oc), fa


def brute_force_knng(data, k: int, queries=None, device: int = 0):
    """brute_force_knng (oracle.hpp:92-127) on the GPU: (ids, float64 dists),
    rows sorted by (distance, id); `queries` restricts the rows computed."""
    data = _as_data(data)
    n, d = data.shape
    if queries is None:
        ids = np.zeros((n, k), np.uint32)
        dd = np.zeros((n, k), np.float64)
        check(N.lib().knng_cuda_bruteforce_knng(data, n, d, k, ids, dd, device))
        return ids, dd
    q = np.ascontiguousarray(queries, dtype=np.uint32)
    ids = np.zeros((len(q), k), np.uint32)
    dd = np.zeros((len(q), k), np.float64)
    check(N.lib().knng_cuda_bruteforce_queries(data, n, d, k, q.ctypes.data, len(q), ids, dd,
                                               device))
    return ids, dd


def recall(approx_ids, exact_ids) -> float:
    """recall (oracle.hpp:131-144): fraction of exact (node, id) pairs present."""
    a = np.asarray(approx_ids)
    e = np.asarray(exact_ids)
    if a.shape != e.shape:
        raise InvalidArgument("recall: graph shapes differ")
    hits = 0
    for u in range(a.shape[0]):
        hits += np.isin(a[u], e[u]).sum()
    return hits / float(a.size)


def locality_permutation(ids, dists, device: int = 0):
    """GPU analogue of greedy_cluster (reorder.hpp:22-50): (sigma, sigma_inv)."""
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    n, k = ids.shape
    sigma = np.zeros(n, np.uint32)
    sigma_inv = np.zeros(n, np.uint32)
    check(N.lib().knng_cuda_locality_permutation(n, k, ids, np.ascontiguousarray(dists, np.float32),
                                                 sigma, sigma_inv, device))
    return sigma, sigma_inv


def scaling_exponent(sizes, evals) -> float:
    """Least-squares slope of log(dist_evals) against log(n)
    (oracle.hpp:147-171), with the reference's argument checks."""
    sizes = [float(s) for s in sizes]
    evals = [float(e) for e in evals]
    if len(sizes) != len(evals) or len(sizes) < 3:
        raise InvalidArgument("scaling_exponent: need at least 3 matched points")
    for i, (s, e) in enumerate(zip(sizes, evals)):
        if s <= 0 or e <= 0:
            raise InvalidArgument("scaling_exponent: sizes and counts must be positive")
        if i > 0 and s <= sizes[i - 1]:
            raise InvalidArgument("scaling_exponent: sizes must be increasing")
    x = np.log(np.asarray(sizes))
    y = np.log(np.asarray(evals))
    dx = x - x.mean()
    return float((dx * (y - y.mean())).sum() / (dx * dx).sum())


def window_cluster_fraction(labels, sigma, window: int = 2000):
    """window_cluster_fraction (reorder.hpp:61-86) of a permutation sigma
    (point i moved to position sigma[i]): for windows of `window` consecutive
    positions, starts advancing by window / 4 with n - window always included,
    the fraction of each cluster.  Returns (window_start, cluster, fraction)
    rows in the reference's order."""
    labels = np.asarray(labels, dtype=np.int64)
    sigma = np.asarray(sigma, dtype=np.int64)
    n = len(sigma)
    if len(labels) != n:
        raise InvalidArgument("window_cluster_fraction: labels/permutation size mismatch")
    if window == 0 or n < window:
        raise InvalidArgument("window_cluster_fraction: window larger than dataset")
    inv = np.empty(n, np.int64)
    inv[sigma] = np.arange(n)
    c = int(labels.max()) + 1 if n else 0
    step = max(1, window // 4)
    out, p = [], 0
    while True:
        cnt = np.bincount(labels[inv[p:p + window]], minlength=c)
        out.extend((p, cl, cnt[cl] / window) for cl in range(c))
        if p == n - window:
            break
        p = min(p + step, n - window)
    return out
