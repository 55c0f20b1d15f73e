"""Join-kernel pass statistics per iteration (diagnostics build only):
    KNNG_CUDA_LIB=scripts/libknng_cuda_stats.so python scripts/join_stats.py C2
"""
import ctypes as C
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2112_06630_b200 as kg
from paper_2112_06630_b200 import _native as N, datasets

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = datasets.CONFIGS[name]
data = datasets.generate(cfg)
fn = N.lib().knng_cuda_debug_join_stats
fn.argtypes = [C.POINTER(C.c_ulonglong)]
buf = (C.c_ulonglong * 8)()
prev = np.zeros(8, np.int64)
print("iter batches nodes passes tiles/pass blocks/pass slabsteps tiles_listed", flush=True)
for it in range(1, 17):
    fn(buf)  # clear
    res = kg.run(data, kg.RunParams(k=cfg.k, max_candidates=cfg.cap, max_iterations=it))
    fn(buf)
    cur = np.array(buf[:], np.int64)
    d = cur - prev
    prev = cur
    if d[0] == 0:
        continue
    p = max(d[2], 1)
    print(it, d[0], d[1], d[2], round(d[3] / p, 2), round(d[4] / p, 2), d[5], d[6], flush=True)
