"""TEST INFRASTRUCTURE ONLY — the CPU checker.

ctypes front-end over the two CPU oracles built by ``oracle/Makefile``:

* ``restated`` -> ``oracle/lib/libknng_oracle.so``: the plain-C restatement
  (``knng_oracle.c``), always buildable from this repo;
* ``reference`` -> ``oracle/_ref/libknng_ref.so``: the unmodified reference
  headers behind ``ref_harness.cpp`` (built only where /root/reference exists;
  the prebuilt .so travels to the GPU box).

Both export the same signatures (prefix ``oracle_`` / ``ref_``), so one wrapper
class serves both.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / reference leg may import this package, and only
as the checker — the product (``paper_2112_06630_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "restated": (os.path.join(HERE, "lib", "libknng_oracle.so"), "oracle_"),
    "reference": (os.path.join(HERE, "_ref", "libknng_ref.so"), "ref_"),
    "reference_native": (os.path.join(HERE, "_ref", "libknng_ref_native.so"), "ref_"),
}

# gcc -m<ext> option -> /proc/cpuinfo flag, for the extensions -march=native
# may have enabled (the rest of the options are tuning, not ISA)
_ISA_FLAG = {
    "-mavx": "avx", "-mavx2": "avx2", "-mfma": "fma", "-mbmi": "bmi1", "-mbmi2": "bmi2",
    "-mf16c": "f16c", "-mavx512f": "avx512f", "-mavx512bw": "avx512bw",
    "-mavx512cd": "avx512cd", "-mavx512dq": "avx512dq", "-mavx512vl": "avx512vl",
    "-mavx512vnni": "avx512_vnni", "-mavx512vbmi": "avx512vbmi", "-mavx512vbmi2": "avx512_vbmi2",
    "-mavx512ifma": "avx512ifma", "-mavx512bitalg": "avx512_bitalg",
    "-mavx512vpopcntdq": "avx512_vpopcntdq", "-mavx512bf16": "avx512_bf16",
    "-mavx512fp16": "avx512_fp16", "-mamx-tile": "amx_tile", "-mamx-bf16": "amx_bf16",
    "-mamx-int8": "amx_int8", "-mavxvnni": "avx_vnni", "-msse4.2": "sse4_2", "-mpopcnt": "popcnt",
    "-mlzcnt": "abm", "-mmovbe": "movbe", "-madx": "adx", "-msha": "sha_ni", "-mvaes": "vaes",
    "-mvpclmulqdq": "vpclmulqdq", "-mgfni": "gfni",
}


def native_compatible() -> tuple:
    """(ok, missing): does this host have every ISA extension the
    -march=native reference build enabled on the build machine?"""
    isa = os.path.join(HERE, "_ref", "native_isa.txt")
    if not (os.path.exists(LIBS["reference_native"][0]) and os.path.exists(isa)):
        return False, ["native build absent"]
    try:
        flags = set()
        for line in open("/proc/cpuinfo"):
            if line.startswith("flags"):
                flags = set(line.split(":", 1)[1].split())
                break
    except OSError:
        return False, ["no /proc/cpuinfo"]
    need = [_ISA_FLAG[o] for o in open(isa).read().split() if o in _ISA_FLAG]
    missing = [f for f in need if f not in flags]
    return not missing, missing


def reference_kind() -> str:
    """The reference build to time: the -march=native one (the reference's own
    CMake flags) when this host supports it, else the portable one."""
    return "reference_native" if native_compatible()[0] else "reference"


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"

u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def build(kind: str = "all") -> None:
    """Build the oracle libraries (make -C oracle <target>)."""
    target = {"all": "all", "restated": "restated", "reference": "ref"}[kind]
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind][0])


class OracleError(RuntimeError):
    pass


class OracleInvalidArgument(ValueError):
    pass


@dataclass
class Graph:
    """Graph rows in the reference's internal heap order."""
    ids: np.ndarray      # (n, k) uint32
    dists: np.ndarray    # (n, k) float32
    flags: np.ndarray    # (n, k) uint8 (1 = is_new)
    rev_deg: Optional[np.ndarray] = None  # (n,) uint32


@dataclass
class Cands:
    ids: np.ndarray         # (n, 2*cap) uint32, new block then old block
    new_counts: np.ndarray  # (n,) uint32
    old_counts: np.ndarray  # (n,) uint32


@dataclass
class RunOut:
    graph: Graph
    iter_evals: np.ndarray
    iter_changes: np.ndarray
    iter_wall: np.ndarray
    total_wall: float
    sigma: Optional[np.ndarray]

    @property
    def total_evals(self) -> int:
        return int(self.iter_evals.sum())

    @property
    def iterations(self) -> int:
        return len(self.iter_evals) - 1


class Oracle:
    def __init__(self, kind: str):
        path, prefix = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; run make -C oracle")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.p = prefix
        L = self.lib
        sz = C.c_uint32
        fn = self._fn
        fn("last_error", C.c_char_p, [])
        fn("run", C.c_int, [f32p, sz, sz, sz, sz, C.c_double, sz, C.c_int, sz, C.c_uint64,
                            u32p, f32p, u8p, u64p, u64p, f64p, u32p, f64p, C.c_void_p])
        fn("capture_step", C.c_int, [f32p, sz, sz, sz, sz, C.c_uint64, sz, u32p, f32p, u8p,
                                     u32p, u32p, u32p, u32p, u32p, f32p, u8p, u32p, u64p, u64p])
        fn("compute_step", C.c_int, [f32p, sz, sz, sz, sz, u32p, f32p, u8p, u32p, u32p, u32p,
                                     C.c_int, u32p, f32p, u8p, u32p, u64p, u64p])
        fn("init_random", C.c_int, [f32p, sz, sz, sz, C.c_uint64, u32p, f32p, u8p, u32p, u64p])
        fn("select_turbo", C.c_int, [sz, sz, sz, u32p, f32p, u8p, C.c_uint64, u32p, u32p, u32p,
                                     u8p])
        fn("brute_force", C.c_int, [f32p, sz, sz, sz, u32p, f64p])
        fn("recall", C.c_int, [sz, sz, u32p, f32p, u32p, f64p])
        fn("greedy_cluster", C.c_int, [sz, sz, u32p, f32p, u8p, u32p, u32p])
        fn("l2_sq", C.c_float, [f32p, f32p, sz])
        fn("block_l2_sq", C.c_int, [f32p, sz, f32p, sz, sz, f32p])
        fn("mutual_block", C.c_int, [f32p, sz, sz, f32p, C.c_void_p, u64p])
        fn("mt64_stream", None, [C.c_uint64, u64p, sz])
        del L

    def _fn(self, name, restype, argtypes):
        f = getattr(self.lib, self.p + name)
        f.restype = restype
        f.argtypes = argtypes
        setattr(self, "_" + name, f)

    def _check(self, rc: int) -> None:
        if rc == 0:
            return
        msg = self._last_error().decode()
        if rc == 1:
            raise OracleInvalidArgument(msg)
        raise OracleError(msg)

    # ---------------------------------------------------------------- API
    def run(self, data, k=20, cap=50, delta=0.001, max_iterations=30, reorder=False,
            reorder_after=1, seed=0) -> RunOut:
        data = np.ascontiguousarray(data, dtype=np.float32)
        n, d = data.shape
        ids = np.zeros((n, k), np.uint32)
        dists = np.zeros((n, k), np.float32)
        flags = np.zeros((n, k), np.uint8)
        ev = np.zeros(max_iterations + 1, np.uint64)
        ch = np.zeros(max_iterations + 1, np.uint64)
        wall = np.zeros(max_iterations + 1, np.float64)
        rows = np.zeros(1, np.uint32)
        total = np.zeros(1, np.float64)
        sigma = np.zeros(n, np.uint32) if reorder else None
        self._check(self._run(data, n, d, k, cap, delta, max_iterations, int(reorder),
                              reorder_after, seed, ids, dists, flags, ev, ch, wall, rows, total,
                              sigma.ctypes.data if sigma is not None else None))
        r = int(rows[0])
        return RunOut(Graph(ids, dists, flags), ev[:r], ch[:r], wall[:r], float(total[0]), sigma)

    def capture_step(self, data, k, cap, seed, t):
        """State of iteration t's join (after select+flag) and the reference result."""
        data = np.ascontiguousarray(data, dtype=np.float32)
        n, d = data.shape
        gi = Graph(np.zeros((n, k), np.uint32), np.zeros((n, k), np.float32),
                   np.zeros((n, k), np.uint8), np.zeros(n, np.uint32))
        go = Graph(np.zeros((n, k), np.uint32), np.zeros((n, k), np.float32),
                   np.zeros((n, k), np.uint8), np.zeros(n, np.uint32))
        c = Cands(np.zeros((n, 2 * cap), np.uint32), np.zeros(n, np.uint32),
                  np.zeros(n, np.uint32))
        changes = np.zeros(1, np.uint64)
        evals = np.zeros(1, np.uint64)
        self._check(self._capture_step(data, n, d, k, cap, seed, t, gi.ids, gi.dists, gi.flags,
                                       gi.rev_deg, c.ids, c.new_counts, c.old_counts, go.ids,
                                       go.dists, go.flags, go.rev_deg, changes, evals))
        return gi, c, go, int(changes[0]), int(evals[0])

    def compute_step(self, data, g: Graph, c: Cands, flat=False):
        data = np.ascontiguousarray(data, dtype=np.float32)
        n, d = data.shape
        k = g.ids.shape[1]
        cap = c.ids.shape[1] // 2
        go = Graph(np.zeros((n, k), np.uint32), np.zeros((n, k), np.float32),
                   np.zeros((n, k), np.uint8), np.zeros(n, np.uint32))
        changes = np.zeros(1, np.uint64)
        evals = np.zeros(1, np.uint64)
        self._check(self._compute_step(
            data, n, d, k, cap, np.ascontiguousarray(g.ids), np.ascontiguousarray(g.dists),
            np.ascontiguousarray(g.flags), np.ascontiguousarray(c.ids),
            np.ascontiguousarray(c.new_counts), np.ascontiguousarray(c.old_counts), int(flat),
            go.ids, go.dists, go.flags, go.rev_deg, changes, evals))
        return go, int(changes[0]), int(evals[0])

    def init_random(self, data, k, seed):
        data = np.ascontiguousarray(data, dtype=np.float32)
        n, d = data.shape
        g = Graph(np.zeros((n, k), np.uint32), np.zeros((n, k), np.float32),
                  np.zeros((n, k), np.uint8), np.zeros(n, np.uint32))
        evals = np.zeros(1, np.uint64)
        self._check(self._init_random(data, n, d, k, seed, g.ids, g.dists, g.flags, g.rev_deg,
                                      evals))
        return g, int(evals[0])

    def select_turbo(self, g: Graph, cap, seed):
        n, k = g.ids.shape
        c = Cands(np.zeros((n, 2 * cap), np.uint32), np.zeros(n, np.uint32),
                  np.zeros(n, np.uint32))
        flags_after = np.zeros((n, k), np.uint8)
        self._check(self._select_turbo(n, k, cap, np.ascontiguousarray(g.ids),
                                       np.ascontiguousarray(g.dists),
                                       np.ascontiguousarray(g.flags), seed, c.ids, c.new_counts,
                                       c.old_counts, flags_after))
        return c, flags_after

    def brute_force(self, data, k):
        data = np.ascontiguousarray(data, dtype=np.float32)
        n, d = data.shape
        ids = np.zeros((n, k), np.uint32)
        dists = np.zeros((n, k), np.float64)
        self._check(self._brute_force(data, n, d, k, ids, dists))
        return ids, dists

    def recall(self, approx_ids, exact_ids) -> float:
        approx_ids = np.ascontiguousarray(approx_ids, dtype=np.uint32)
        n, k = approx_ids.shape
        out = np.zeros(1, np.float64)
        self._check(self._recall(n, k, approx_ids, np.zeros((n, k), np.float32),
                                 np.ascontiguousarray(exact_ids, dtype=np.uint32), out))
        return float(out[0])

    def greedy_cluster(self, g: Graph):
        n, k = g.ids.shape
        sigma = np.zeros(n, np.uint32)
        sigma_inv = np.zeros(n, np.uint32)
        self._check(self._greedy_cluster(n, k, np.ascontiguousarray(g.ids),
                                         np.ascontiguousarray(g.dists),
                                         np.ascontiguousarray(g.flags), sigma, sigma_inv))
        return sigma, sigma_inv

    def l2_sq(self, a, b) -> float:
        a = np.ascontiguousarray(a, dtype=np.float32)
        b = np.ascontiguousarray(b, dtype=np.float32)
        return float(self._l2_sq(a, b, a.shape[0]))

    def block_l2_sq(self, rows_a, rows_b):
        rows_a = np.ascontiguousarray(rows_a, dtype=np.float32)
        rows_b = np.ascontiguousarray(rows_b, dtype=np.float32)
        out = np.zeros(rows_a.shape[0] * rows_b.shape[0], np.float32)
        self._check(self._block_l2_sq(rows_a, rows_a.shape[0], rows_b, rows_b.shape[0],
                                      rows_a.shape[1], out))
        return out.reshape(rows_a.shape[0], rows_b.shape[0])

    def mutual_block(self, rows):
        rows = np.ascontiguousarray(rows, dtype=np.float32)
        m, d = rows.shape
        mat = np.zeros((m, m), np.float32)
        visits = np.zeros(max(1, m * (m - 1)), np.uint32)
        count = np.zeros(1, np.uint64)
        self._check(self._mutual_block(rows, m, d, mat, visits.ctypes.data, count))
        cnt = int(count[0])
        return mat, visits[: 2 * cnt].reshape(cnt, 2)

    def mt64_stream(self, seed, count):
        out = np.zeros(count, np.uint64)
        self._mt64_stream(seed, out, count)
        return out


_cache: dict = {}


def load(kind: str = "restated") -> Oracle:
    if kind not in _cache:
        _cache[kind] = Oracle(kind)
    return _cache[kind]
