"""B200-native NN-Descent (squared L2) — GPU K-NNG construction.

The product is the CUDA library ``lib/libknng_cuda.so`` (C-ABI in
``include/knng_cuda.h``); :mod:`.knng` mirrors the reference's knng
interface on top of it.  Build with ``python -m paper_2112_06630_b200.build``.
"""
from .knng import (  # noqa: F401
    CandidateSet, InvalidArgument, IterationMetrics, KnnGraph, KnngCudaError, RunMetrics,
    RunParams, RunResult, brute_force_knng, candidate_distances, compute_step, device_count,
    flop_count, init_random, locality_permutation, nndescent_l2, recall, run, run_device,
    run_multi,
    scaling_exponent, select_turbo, window_cluster_fraction,
)
