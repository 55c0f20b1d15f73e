"""Build join-kernel variants (scripts/libknng_cuda_<tag>.so) for A/B timing.

    python scripts/build_variants.py tag:-DKNNG_JOIN_STAGES=4,-DKNNG_JOIN_PASSBLK=11 ...
    python scripts/build_variants.py tag@join_tc.cu:-DKNNG_TC_PROF=1   (another source file)
Run a variant with KNNG_CUDA_LIB=scripts/libknng_cuda_<tag>.so.
"""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_06630_b200 import build as B

B.build()
for spec in sys.argv[1:]:
    tag, flags = spec.split(":", 1)
    src = "join.cu"
    if "@" in tag:
        tag, src = tag.split("@")
    objs = [os.path.join(B.OBJ, s.replace(".cu", ".o")) for s in B.SOURCES if s != src]
    o = os.path.join(B.OBJ, f"{src[:-3]}_{tag}.o")
    subprocess.run([B.nvcc(), *B.ARCH, *B.FLAGS, *B.PER_FILE.get(src, []), *flags.split(","),
                    "-c", os.path.join(B.CSRC, src), "-o", o], check=True)
    lib = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"libknng_cuda_{tag}.so")
    subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", lib, *objs, o, "-cudart", "static"], check=True)
    print(lib)
