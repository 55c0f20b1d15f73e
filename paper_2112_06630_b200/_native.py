"""ctypes binding of libknng_cuda.so (C-ABI: include/knng_cuda.h).

The shared library is the product; this module only declares its symbols.
Loading fails loudly when the library is missing — there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KNNG_CUDA_LIB") or os.path.join(PKG, "lib", "libknng_cuda.so")

OK = 0
INVALID_ARGUMENT = 1
CUDA_ERROR = 2
NCCL_ERROR = 3
OUT_OF_MEMORY = 4
NOT_IMPLEMENTED = 5

MAX_K = 32
MAX_CANDIDATES = 64

KERNEL_NAMES = ("init", "degree", "sample", "finalize", "join", "reorder", "merge", "index")

# every symbol include/knng_cuda.h declares
EXPORTS = (
    "knng_cuda_params_default",
    "knng_cuda_last_error",
    "knng_cuda_device_count",
    "knng_cuda_nndescent_l2",
    "knng_cuda_run",
    "knng_cuda_run_device",
    "knng_cuda_local_join",
    "knng_cuda_candidate_distances",
    "knng_cuda_init_random",
    "knng_cuda_select",
    "knng_cuda_bruteforce_knng",
    "knng_cuda_bruteforce_queries",
    "knng_cuda_locality_permutation",
    "knng_cuda_shard_create",
    "knng_cuda_shard_destroy",
    "knng_cuda_seed_sequence",
    "knng_cuda_shard_init",
    "knng_cuda_shard_degree",
    "knng_cuda_shard_sample",
    "knng_cuda_shard_offers",
    "knng_cuda_shard_step",
    "knng_cuda_shard_merge",
    "knng_cuda_shard_export",
    "knng_cuda_shard_metrics",
    "knng_cuda_shard_reorder",
    "knng_cuda_run_multi",
)


class ShardInfo(C.Structure):
    _fields_ = [
        ("keys", C.c_void_p),
        ("flags", C.c_void_p),
        ("maxd", C.c_void_p),
        ("indeg", C.c_void_p),
        ("rows_alloc", C.c_uint32),
        ("chunk", C.c_uint32),
        ("lo", C.c_uint32),
        ("hi", C.c_uint32),
        ("stream", C.c_void_p),
        ("seg_cap", C.c_uint64),
    ]


class Params(C.Structure):
    _fields_ = [
        ("k", C.c_uint32),
        ("max_candidates", C.c_uint32),
        ("termination_delta", C.c_double),
        ("max_iterations", C.c_uint32),
        ("reorder", C.c_int32),
        ("reorder_after_iteration", C.c_uint32),
        ("seed", C.c_uint64),
        ("device", C.c_int32),
        ("profile", C.c_int32),
        ("deterministic", C.c_int32),
        ("observer", C.c_void_p),
        ("observer_user", C.c_void_p),
    ]


# knng_cuda_observer_fn
OBSERVER = C.CFUNCTYPE(None, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32),
                       C.POINTER(C.c_float), C.POINTER(C.c_uint8), C.c_void_p)


class Iteration(C.Structure):
    _fields_ = [
        ("iteration", C.c_uint32),
        ("wall_time_s", C.c_double),
        ("dist_evals", C.c_uint64),
        ("changes", C.c_uint64),
        ("join_candidates", C.c_uint64),
        ("join_ms", C.c_double),
    ]


class Metrics(C.Structure):
    _fields_ = [
        ("iterations", C.POINTER(Iteration)),
        ("capacity", C.c_uint32),
        ("n_rows", C.c_uint32),
        ("total_wall_time_s", C.c_double),
        ("total_dist_evals", C.c_uint64),
        ("total_changes", C.c_uint64),
        ("kernel_ms", C.c_double * 8),
        ("kernel_launches", C.c_uint64 * 8),
        ("join_candidates", C.c_uint64),
        ("join_evals", C.c_uint64),
        ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64),
    ]


u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
vp = C.c_void_p
u32 = C.c_uint32

_lib = None


def lib() -> C.CDLL:
    """The loaded product library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2112_06630_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)

    def fn(name, restype, argtypes):
        f = getattr(L, name)
        f.restype = restype
        f.argtypes = argtypes

    fn("knng_cuda_params_default", None, [C.POINTER(Params)])
    fn("knng_cuda_last_error", C.c_char_p, [])
    fn("knng_cuda_device_count", C.c_int, [])
    fn("knng_cuda_nndescent_l2", C.c_int, [f32p, u32, u32, u32, C.c_double, C.c_double,
                                           C.c_uint64, u32, C.c_int, u32p, f32p,
                                           C.POINTER(Metrics)])
    fn("knng_cuda_run", C.c_int, [vp, u32, u32, C.POINTER(Params), vp, vp, vp, vp,
                                  C.POINTER(Metrics)])
    fn("knng_cuda_run_device", C.c_int, [vp, u32, u32, C.POINTER(Params), vp, vp,
                                         C.POINTER(Metrics), vp])
    fn("knng_cuda_local_join", C.c_int, [f32p, u32, u32, u32, u32, u32p, f32p, u8p, u32p, u32p,
                                         u32p, u32p, f32p, u8p, u32p, u64p, u64p, C.c_int])
    fn("knng_cuda_candidate_distances", C.c_int, [f32p, u32, u32, u32, u32p, u32p, u32p, u64p,
                                                  f32p, C.c_uint64, C.c_int])
    fn("knng_cuda_init_random", C.c_int, [f32p, u32, u32, u32, C.c_uint64, u32p, f32p, u8p,
                                          u32p, u64p, C.c_int])
    fn("knng_cuda_select", C.c_int, [u32, u32, u32, u32p, f32p, u8p, C.c_uint64, u32p, u32p,
                                     u32p, u8p, C.c_int])
    fn("knng_cuda_bruteforce_knng", C.c_int, [f32p, u32, u32, u32, u32p, f64p, C.c_int])
    fn("knng_cuda_bruteforce_queries", C.c_int, [f32p, u32, u32, u32, vp, u32, u32p, f64p,
                                                 C.c_int])
    fn("knng_cuda_locality_permutation", C.c_int, [u32, u32, u32p, f32p, u32p, u32p, C.c_int])
    fn("knng_cuda_shard_create", C.c_int, [vp, u32, u32, C.POINTER(Params), u32, u32, vp,
                                           C.POINTER(vp), C.POINTER(ShardInfo)])
    fn("knng_cuda_shard_destroy", C.c_int, [vp])
    fn("knng_cuda_seed_sequence", None, [C.c_uint64, u32, u64p])
    fn("knng_cuda_shard_init", C.c_int, [vp, C.c_uint64])
    fn("knng_cuda_shard_degree", C.c_int, [vp])
    fn("knng_cuda_shard_sample", C.c_int, [vp, C.c_uint64, u64p, C.POINTER(vp)])
    fn("knng_cuda_shard_offers", C.c_int, [vp, vp, C.c_uint64])
    fn("knng_cuda_shard_step", C.c_int, [vp, u64p, u64p, C.POINTER(vp)])
    fn("knng_cuda_shard_merge", C.c_int, [vp, vp, C.c_uint64, u64p])
    fn("knng_cuda_shard_export", C.c_int, [vp, vp, vp])
    fn("knng_cuda_shard_metrics", C.c_int, [vp, C.POINTER(Metrics)])
    fn("knng_cuda_shard_reorder", C.c_int, [vp, C.POINTER(ShardInfo), C.POINTER(vp),
                                            C.POINTER(vp)])
    fn("knng_cuda_run_multi", C.c_int, [f32p, u32, u32, C.POINTER(Params), C.c_int, vp, u32p,
                                        f32p, C.POINTER(Metrics)])
    _lib = L
    return L


class KnngCudaError(RuntimeError):
    """CUDA / NCCL / allocation failure inside libknng_cuda (codes 2-5)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class InvalidArgument(ValueError):
    """The reference's std::invalid_argument cases (code 1)."""


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().knng_cuda_last_error().decode(errors="replace")
    if rc == INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    raise KnngCudaError(rc, msg)
