"""Per-phase clock totals of the tcgen05 byte join (diagnostics build):
    KNNG_CUDA_LIB=scripts/libknng_cuda_tcprof.so KNNG_U8_TC=1 python scripts/u8tc_prof.py
"""
import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2112_06630_b200 as kg
from paper_2112_06630_b200 import _native as N, datasets
cfg = datasets.CONFIGS["C2"]
data = datasets.generate(cfg)
fn = N.lib().knng_cuda_debug_u8tc_prof
buf = (C.c_ulonglong * 8)()
fn(buf)
kg.run(data, kg.RunParams(k=cfg.k, max_candidates=cfg.cap, max_iterations=1))
fn(buf)
names = ["meta", "tma_issue", "wait_rows", "mma_issue", "mma_wait", "epilogue"]
tot = sum(buf[:6])
print({n: round(buf[i] / 148 / 1.965e3, 1) for i, n in enumerate(names)}, "us per SM (iteration 1)")
