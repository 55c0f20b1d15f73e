"""The C-ABI library builds, loads and exports exactly what include/knng_cuda.h
declares; parameter errors map to the reference's std::invalid_argument cases;
with no GPU every compute entry fails loudly (there is no CPU path)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "knng_cuda.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(knng_cuda_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_binding_list():
    from paper_2112_06630_b200 import _native
    assert declared_symbols() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol(native):
    for name in declared_symbols():
        assert hasattr(native, name), name


def test_library_is_sm100a_only(native):
    import subprocess
    from paper_2112_06630_b200 import _native
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for arch in ("sm_80", "sm_90", "sm_103"):
        assert arch not in out.replace("sm_100a", "")


def test_params_default_match_reference(native):
    from paper_2112_06630_b200 import _native
    p = _native.Params()
    native.knng_cuda_params_default(C.byref(p))
    # RunParams defaults (descent.hpp:18-28)
    assert (p.k, p.max_candidates, p.termination_delta, p.max_iterations, p.reorder,
            p.reorder_after_iteration, p.seed) == (20, 50, 0.001, 30, 0, 1, 0)


def test_invalid_arguments_before_any_device_work(native):
    import paper_2112_06630_b200 as kg
    data = np.random.default_rng(0).standard_normal((30, 8), dtype=np.float32)
    # test_descent.cpp:12-27
    for params in (kg.RunParams(k=1), kg.RunParams(termination_delta=0.0),
                   kg.RunParams(k=20, max_candidates=19), kg.RunParams(k=30, max_candidates=50)):
        with pytest.raises(kg.InvalidArgument):
            kg.run(data, params)
    with pytest.raises(kg.InvalidArgument):
        kg.nndescent_l2(data, k=10, sample_rate=0.5)  # cap 5 < k
    # caller-owned result arrays must match the graph's shape and types
    p = kg.RunParams(k=5, max_candidates=10)
    good = (np.zeros((30, 5), np.uint32), np.zeros((30, 5), np.float32), np.zeros((30, 5), np.uint8))
    for bad in ((np.zeros((30, 4), np.uint32),) + good[1:],
                (good[0].astype(np.int64),) + good[1:],
                (good[0], np.zeros((5, 30), np.float32).T, good[2]),   # not C-contiguous
                good[:2] + (np.zeros((30, 5), np.float32),)):
        with pytest.raises(kg.InvalidArgument):
            kg.run(data, p, out=kg.KnnGraph(*bad))


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES") is None and
                    os.path.exists("/dev/nvidia0"), reason="a GPU is present")
def test_no_gpu_fails_loudly(native):
    import paper_2112_06630_b200 as kg
    if kg.device_count() > 0:
        pytest.skip("GPU present")
    data = np.random.default_rng(0).standard_normal((100, 8), dtype=np.float32)
    with pytest.raises(kg.KnngCudaError):
        kg.run(data, kg.RunParams(k=5, max_candidates=10))


DROPIN = os.path.join(ROOT, "tests", "cpp", "build", "dropin_check")


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"),
                    reason="reference headers absent")
def test_cpp_dropin_builds_against_reference_headers(native):
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    out = subprocess.run([DROPIN], capture_output=True, text=True)
    # no GPU here: the wrapper must fail loudly with std::runtime_error (rc 3),
    # after mapping the parameter error to std::invalid_argument
    assert out.returncode in (0, 3), out.stdout + out.stderr
    assert out.stdout.startswith("dropin ")


@pytest.mark.gpu
def test_cpp_dropin_on_gpu(gpu):
    import subprocess
    if not os.path.exists(DROPIN):
        pytest.skip("drop-in check not built (needs the reference headers at build time)")
    out = subprocess.run([DROPIN], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "dropin OK" in out.stdout, out.stdout + out.stderr
