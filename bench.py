#!/usr/bin/env python
"""Benchmark: GPU NN-Descent K-NNG build (squared L2) — BASELINE.json's metric
"K-NNG build time & distance evals/s at matched recall@k vs CPU ref".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2]

A step is one complete K-NNG build (knng::run: random init + iterations to
termination) of the config's synthetic dataset.  Default workload: config C5
(BASELINE.json configs[4], n=1,000,000 x d=960 L2-normalised Gamma features,
k=20, cap 50): BASELINE.json quotes its metric on no single config, so the
line is the largest single-GPU config (by data and by distance work).

`value` = distance evaluations per second over the K timed builds, whole job,
inputs resident in HBM (device-pointer entry knng_cuda_run_device), device
time from CUDA events, max over ranks.  `e2e` = the same metric through the
host-pointer C-ABI (knng_cuda_run) with the pinned-host -> device copy of the
data and the device -> host copy of the graph inside every step.
`--impl reference` times the reference's own CPU code (oracle/_ref, the
unmodified knng headers built with the reference's own -march=native Release
flags when the host supports them) on the host.  knng::run is single-threaded
by contract, so the arm runs one independent build per host
core concurrently, each on its own bounded slice of the config's rows, and
reports their summed evaluations over the step's wall time (all the host
threads it can use).  With N > 1 (torchrun) one build is sharded over the N
GPUs (paper_2112_06630_b200/shard.py).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2112_06630_b200 import datasets  # noqa: E402

METRIC = "dist_evals_per_s"
UNIT = "distance evaluations/s"
PROFILE_TRAFFIC = os.path.join(ROOT, "profiles", "join_traffic.json")


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.25)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for r in csv.reader(f):
                if len(r) >= 9:
                    rows.append([x.strip() for x in r])
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def ffma_peak_tflops(device: int):
    import ctypes as C
    path = os.path.join(ROOT, "paper_2112_06630_b200", "lib", "libknng_diag.so")
    if not os.path.exists(path):
        return None
    lib = C.CDLL(path)
    t = C.c_double(0)
    t2 = C.c_double(0)
    ms = C.c_double(0)
    if lib.knng_diag_ffma_peak(device, C.byref(t), C.byref(ms)) != 0:
        return None
    if lib.knng_diag_ffma2_peak(device, C.byref(t2)) != 0:
        t2.value = 0.0
    return max(t.value, t2.value)


def imma_peak_tops(device: int):
    """Measured legacy integer MMA peak (mma.sync m16n8k32 u8, TOPS)."""
    import ctypes as C
    path = os.path.join(ROOT, "paper_2112_06630_b200", "lib", "libknng_diag.so")
    if not os.path.exists(path):
        return None
    lib = C.CDLL(path)
    t = C.c_double(0)
    if not hasattr(lib, "knng_diag_imma_peak") or lib.knng_diag_imma_peak(device, C.byref(t)) != 0:
        return None
    return t.value


def byte_valued(data) -> bool:
    """Does the build take the byte-valued join (csrc/join_u8.cu)?  Same rule
    as the library: every coordinate an integer in [0, 255], stride / 8 <= 258,
    and KNNG_JOIN_U8 not set to 0."""
    if os.environ.get("KNNG_JOIN_U8", "1").startswith("0"):
        return False
    stride = (data.shape[1] + 7) // 8 * 8
    return bool(stride // 8 <= 258 and np.all((data >= 0) & (data <= 255) & (data == np.rint(data))))


def u8_roofline(mets, n, d, k, imma_tops, fp32_tflops, config):
    """Roofline of the byte-valued join kernel (join_u8_kernel).

    Per launch: Q = sum_u (nn_u + no_u) * (8 Kl + 32 + 8) + 12 n k bytes (the
    byte rows with Kl = ceil64(stride / 8) bytes per reference lane, the 8
    lane norms, id and row maximum per listed candidate, the graph) and
    F = evals * 2 d integer ops (the per-lane dot products); t* =
    max(F / pi_imma, Q / beta_hbm), frac = sum(t*) / sum(t).  The byte copy
    of C2 (70 MB) is L2-resident, so the HBM bound is conservative; ncu's L1
    throughput is the limiter (profiles/README.md).
    """
    stride = (d + 7) // 8 * 8
    kl = (stride // 8 + 63) // 64 * 64
    beta, beta_src = 6650.0, "fallback 6650 GB/s (B200_PROFILING.md)"
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        beta = float(json.load(open(mp))["hbm_gbs"])
        beta_src = "MEASURED_PEAKS.json hbm_gbs (measured)"
    pi = imma_tops or 500.0
    pi_src = ("measured mma.sync m16n8k32 u8 microbenchmark (libknng_diag), this box" if imma_tops
              else "fallback 500 TOPS")
    F = Q = t = t_star = t_int = t_hbm = E = 0.0
    launches = 0
    for m in mets:
        for it in m.iterations:
            if it.iteration == 0 or it.join_ms <= 0:
                continue
            f = it.dist_evals * 2.0 * d
            q = it.join_candidates * (8 * kl + 32 + 8) + 12.0 * n * k
            ti, th = f / (pi * 1e12), q / (beta * 1e9)
            F += f
            Q += q
            E += it.dist_evals
            t += it.join_ms * 1e-3
            t_int += ti
            t_hbm += th
            t_star += max(ti, th)
            launches += 1
    frac = t_star / t if t else 0.0
    traffic, traffic_note = _traffic(config)
    if t_int >= t_hbm:
        roof = {"bound": "tensor", "achieved": round(frac * pi, 2), "peak": round(pi, 1),
                "unit": "TOPS (int8)", "peak_source": pi_src}
    else:
        roof = {"bound": "hbm", "achieved": round(frac * beta, 1), "peak": beta, "unit": "GB/s",
                "peak_source": beta_src}
    roof.update({
        "frac": round(frac, 4), "traffic": traffic, "traffic_note": traffic_note,
        "kernel": "join_u8_kernel (local-join distance stage, byte-valued data: per-lane integer "
                  "dot products on the tensor cores, bit-identical to the reference)",
        "frac_definition": "sum over launches of max(F_int/pi_imma, Q/beta) / sum of launch times",
        "gather_gbs_achieved": round(Q / t / 1e9, 1) if t else None,
        "int_tops_achieved": round(F / t / 1e12, 2) if t else None,
        "fp32_equiv_tflops_achieved": round(E * (3 * d - 1) / t / 1e12, 2) if t else None,
        "fp32_peak_tflops": round(fp32_tflops, 2) if fp32_tflops else None,
        "algorithmic_int_ops_per_launch": int(F / max(1, launches)),
        "algorithmic_bytes_per_launch": int(Q / max(1, launches)),
        "avg_launch_ms": round(t * 1e3 / max(1, launches), 4),
        "launches": launches, "imma_peak_tops": round(pi, 1), "hbm_peak_gbs": beta,
    })
    return roof


def _traffic(config):
    traffic = traffic_note = None
    if os.path.exists(PROFILE_TRAFFIC):
        try:
            tr = json.load(open(PROFILE_TRAFFIC)).get(config)
            if isinstance(tr, dict):
                traffic = tr.get("bytes_per_launch")
                traffic_note = (f"ncu dram bytes of the {tr.get('launch')} launch of "
                                f"{tr.get('kernel', 'the join')}; algorithmic bytes of that launch "
                                f"{tr.get('algorithmic_bytes_same_launch'):.4g} ({tr.get('source')})")
            else:
                traffic = tr
        except (OSError, ValueError, TypeError):
            traffic = None
    return traffic, traffic_note


def join_roofline(mets, n, d, k, peak_tflops, config):
    """Roofline of the local-join distance kernel (join5_kernel, csrc/join5.cu).

    Per launch (one per iteration) the algorithmic work is, after SURVEY.md
    §8d: F = evals * (3d - 1) credited flops (distance.hpp:19-21) and
    Q = sum_u (nn_u + no_u) * (4 * stride + 8) + 12 n k gather bytes.  Its
    roofline time is t* = max(F / pi_fp32, Q / beta_hbm); the reported
    fraction is sum(t*) / sum(t) over every timed launch, so iterations that
    are FP32-bound (early, large lists) and HBM-bound (late) both count.
    """
    stride = (d + 7) // 8 * 8
    beta = 6650.0
    beta_src = "fallback 6650 GB/s (B200_PROFILING.md)"
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        beta = float(json.load(open(mp))["hbm_gbs"])
        beta_src = "MEASURED_PEAKS.json hbm_gbs (measured)"
    pi = peak_tflops or 74.0
    pi_src = ("measured FFMA/FFMA2 microbenchmark (libknng_diag), this box" if peak_tflops
              else "fallback 74 TFLOP/s nominal")
    F = Q = t = t_star = t_fp = t_hbm = 0.0
    launches = 0
    for m in mets:
        for it in m.iterations:
            if it.iteration == 0 or it.join_ms <= 0:
                continue
            f = it.dist_evals * (3 * d - 1)
            q = it.join_candidates * (4 * stride + 8) + 12 * n * k
            tf, th = f / (pi * 1e12), q / (beta * 1e9)
            F += f
            Q += q
            t += it.join_ms * 1e-3
            t_fp += tf
            t_hbm += th
            t_star += max(tf, th)
            launches += 1
    traffic, traffic_note = _traffic(config)
    frac = t_star / t if t else 0.0
    if t_fp >= t_hbm:
        roof = {"bound": "fp32", "achieved": round(frac * pi, 3), "peak": round(pi, 2),
                "unit": "TFLOP/s", "peak_source": pi_src}
    else:
        roof = {"bound": "hbm", "achieved": round(frac * beta, 1), "peak": beta, "unit": "GB/s",
                "peak_source": beta_src}
    roof.update({
        "frac": round(frac, 4), "traffic": traffic, "traffic_note": traffic_note,
        "kernel": "join5_kernel (local-join distance stage, 5 x 10 tiles)",
        "frac_definition": "sum over launches of max(F/pi, Q/beta) / sum of launch times",
        "fp32_tflops_achieved": round(F / t / 1e12, 3) if t else None,
        "gather_gbs_achieved": round(Q / t / 1e9, 1) if t else None,
        "algorithmic_flops_per_launch": int(F / max(1, launches)),
        "algorithmic_bytes_per_launch": int(Q / max(1, launches)),
        "avg_launch_ms": round(t * 1e3 / max(1, launches), 4),
        "launches": launches,
        "fp32_peak_tflops": round(pi, 2), "hbm_peak_gbs": beta,
    })
    return roof


def reference_recall_sample(data, k, cfg, ids_gpu, sample, reference_ids=None):
    """recall@k of the GPU graph on a node sample against the exact K-NNG (GPU
    brute force, index-exact vs the CPU oracle), and the reference's recall on
    the same sample: from a same-run reference build when one was made, else
    from the committed full-config reference build of this config with the
    same seed (tests/golden/reference_rows_<C>.npz, scripts/reference_full.py)."""
    import paper_2112_06630_b200 as kg
    ex, _ = kg.brute_force_knng(data, k, queries=sample)
    out = {"gpu": round(kg.recall(ids_gpu[sample], ex), 5), "sample_nodes": int(len(sample))}
    if reference_ids is not None:
        out["reference"] = round(kg.recall(reference_ids[sample], ex), 5)
        out["reference_source"] = "same-run reference build"
    else:
        path = os.path.join(ROOT, "tests", "golden", f"reference_rows_{cfg.name}.npz")
        if os.path.exists(path):
            z = np.load(path)
            if z["sample"].shape == sample.shape and np.array_equal(z["sample"], sample):
                out["reference"] = round(kg.recall(z["ids"], ex), 5)
                meta = os.path.join(ROOT, "profiles", f"reference_full_{cfg.name}.json")
                src = "committed full-config reference build, same seed and parameters"
                if os.path.exists(meta):
                    mj = json.load(open(meta))
                    src += (f" ({mj['iterations']} iterations, {mj['total_wall_s']:.1f} s on one "
                            f"core of {mj['cpu']}; tests/golden/reference_rows_{cfg.name}.npz)")
                out["reference_source"] = src
    if "reference" in out:
        out["gap_pp"] = round(100.0 * (out["gpu"] - out["reference"]), 3)
    return out


def reference_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


# rows per reference build in the bounded CPU sample (about 5-10 s of one core each)
REF_SAMPLE_ROWS = {"C1": 10_000, "C2": 70_000, "C3": 40_000, "C4": 100_000, "C5": 20_000}


def reference_step(O, data, cfg, rows, threads):
    """One step of the reference arm: `threads` concurrent knng::run builds
    (the reference is single-threaded by contract), build t on rows
    [t*rows, (t+1)*rows) of the workload (wrapping), same k / cap / delta /
    seed.  Returns (evals, wall seconds, iterations per build)."""
    from concurrent.futures import ThreadPoolExecutor
    n = data.shape[0]
    rows = min(rows, n)
    slices = []
    for t in range(threads):
        s = (t * rows) % n
        if s + rows > n:
            s = 0
        slices.append(np.ascontiguousarray(data[s:s + rows]))

    def one(x):
        return O.run(x, k=cfg.k, cap=cfg.cap, delta=cfg.delta, seed=cfg.seed)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        outs = list(ex.map(one, slices))
    wall = time.perf_counter() - t0
    full_ids = outs[0].graph.ids if rows == n else None
    return (sum(r.total_evals for r in outs), wall,
            float(np.mean([r.iterations for r in outs])), full_ids)


def reference_oracle():
    import oracle
    kind = oracle.reference_kind() if oracle.available("reference") else "restated"
    return oracle, kind, oracle.load(kind)


def run_sharded_bench(args, rank, world, local):
    """N > 1: one K-NNG build sharded over the N GPUs (vertex-range ownership,
    NCCL exchanges; paper_2112_06630_b200/shard.py).  Total work is fixed, so
    scaling is strong."""
    import torch
    import torch.distributed as dist

    import paper_2112_06630_b200 as kg
    from paper_2112_06630_b200.shard import GpuShardEngine, gather_graph, run_sharded
    # KNNG_DIST_BACKEND=gloo: the collectives through host memory, so several
    # ranks can share one GPU (a functional check of this path on a one-GPU
    # box; NCCL, the default, needs a GPU per rank)
    backend = os.environ.get("KNNG_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if "RANK" not in os.environ:  # --sharded on one GPU without torchrun
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(29500 + os.getpid() % 1000))
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    cfg = datasets.CONFIGS[args.config]
    data = datasets.generate(cfg)  # same instance on every rank (replicated data)
    n, d = data.shape
    k, cap = cfg.k, cfg.cap
    params = kg.RunParams(k=k, max_candidates=cap, termination_delta=cfg.delta, seed=cfg.seed,
                          device=local, profile=True)
    d_data = torch.from_numpy(data).to(f"cuda:{local}")
    eng = GpuShardEngine(d_data, params, rank, world)
    peak = ffma_peak_tflops(local)
    u8 = byte_valued(data)
    ipeak = imma_peak_tops(local) if u8 else None
    for _ in range(args.warmup):
        run_sharded(eng, params)
    rows_before = len(eng.metrics().iterations)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    results = [run_sharded(eng, params) for _ in range(args.steps)]
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    # this rank's join-kernel roofline over the timed builds (its own share of
    # evaluations, candidates and owned rows)
    shard_m = eng.metrics()
    shard_m.iterations = shard_m.iterations[rows_before:]
    owned = eng.hi - eng.lo
    roof = (u8_roofline([shard_m], owned, d, k, ipeak, peak, args.config) if u8 else
            join_roofline([shard_m], owned, d, k, peak, args.config))
    roof["scope"] = f"rank {rank} of {world}: its join launches and its share of the work"
    evals = sum(r.metrics.total_dist_evals for r in results)  # already summed over ranks
    iters = sum(len(r.metrics.iterations) - 1 for r in results)
    sent = sum(r.bytes_exchanged for r in results)
    # e2e: pinned host data -> device, sharded build, owned rows -> host
    pinned = torch.empty((n, d), dtype=torch.float32, pin_memory=True)
    pinned.numpy()[:] = data
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    e2e_evals = 0
    d2h = 0
    ids_h = dists_h = None  # page-locked result rows, reused
    for _ in range(args.steps):
        dd = pinned.to(f"cuda:{local}", non_blocking=True)
        torch.cuda.synchronize()
        e = GpuShardEngine(dd, params, rank, world)
        r = run_sharded(e, params)
        if ids_h is None or ids_h.shape != r.ids.shape:
            ids_h = torch.empty(r.ids.shape, dtype=r.ids.dtype, pin_memory=True)
            dists_h = torch.empty(r.dists.shape, dtype=r.dists.dtype, pin_memory=True)
        ids_h.copy_(r.ids)
        dists_h.copy_(r.dists)
        d2h += ids_h.numel() * 4 + dists_h.numel() * 4
        e2e_evals += r.metrics.total_dist_evals
        e.close()
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([ms, e2e_s], dtype=torch.float64,
                     device=f"cuda:{local}" if backend == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, e2e_s = float(t[0]), float(t[1])
    out = None
    ids_all, _ = gather_graph(results[-1], n, k)
    if rank == 0:
        sample = np.random.default_rng(1).choice(n, size=min(n, args.recall_sample),
                                                 replace=False).astype(np.uint32)
        rec = reference_recall_sample(data, k, cfg, ids_all.cpu().numpy().astype(np.uint32),
                                      sample)
        out = {
            "metric": METRIC, "value": round(evals / (ms * 1e-3), 1), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.description}", "n": n, "d": d, "k": k,
                       "max_candidates": cap, "delta": cfg.delta, "seed": cfg.seed,
                       "step": "one complete K-NNG build sharded over all GPUs",
                       "l2": "inputs larger than L2 (data %.1f MB > 126 MB)" % (n * d * 4 / 1e6),
                       "parallelism": f"{world} vertex-range shards, replicated data; NCCL "
                                      "all-reduce of in-degree, all-to-all of reverse offers "
                                      "and of proposals, all-gather of row maxima"},
            "build_time_ms": round(ms / args.steps, 3),
            "iterations_per_s": round(iters / (ms * 1e-3), 2),
            "iterations_per_build": round(iters / args.steps, 2),
            "recall_at_k": rec,
            "e2e": {"value": round(e2e_evals / e2e_s, 1), "unit": UNIT,
                    "h2d_bytes_per_step": n * d * 4,
                    "d2h_bytes_per_step": int(d2h / args.steps)},
            "exchange_bytes_per_step_rank0": int(sent / args.steps),
            # per rank and build: init + export, and per iteration partial
            # in-degree, reset, sample, offers, finalize (2), offsets (2 scans),
            # capacity check, reverse scatter, distances, merge (2), export
            # count / scan / bounds / write, received count / scan / scatter /
            # merge
            "gpu_launches": int(2 * args.steps + 21 * iters),
            "roofline": roof,
            "cpu_baseline": None,
            "clocks": clk,
        }
    eng.close()
    dist.barrier()
    dist.destroy_process_group()
    return out


def run_ours(args, rank, world, local):
    import torch
    import paper_2112_06630_b200 as kg
    if world > 1 or args.sharded:
        return run_sharded_bench(args, rank, world, local)
    torch.cuda.set_device(local)
    dist = None

    cfg = datasets.CONFIGS[args.config]
    # replicas: each rank builds its own seeded instance
    cfg_r = datasets.Config(cfg.name, cfg.n, cfg.d, cfg.k, cfg.cap, cfg.delta, cfg.seed + rank,
                            cfg.description)
    data = datasets.generate(cfg_r)
    n, d = data.shape
    k, cap = cfg.k, cfg.cap
    params = kg.RunParams(k=k, max_candidates=cap, termination_delta=cfg.delta, seed=cfg_r.seed,
                          device=local, profile=True)
    peak = ffma_peak_tflops(local)
    u8 = byte_valued(data)
    ipeak = imma_peak_tops(local) if u8 else None

    d_data = torch.from_numpy(data).to(f"cuda:{local}")
    d_ids = torch.empty((n, k), dtype=torch.int32, device=f"cuda:{local}")
    d_dists = torch.empty((n, k), dtype=torch.float32, device=f"cuda:{local}")
    stream = torch.cuda.current_stream().cuda_stream

    def step():
        return kg.run_device(d_data.data_ptr(), n, d, params, d_ids.data_ptr(),
                             d_dists.data_ptr(), stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    mets = [step() for _ in range(args.steps)]
    e1.record()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    evals = sum(m.total_dist_evals for m in mets)
    iters = sum(len(m.iterations) - 1 for m in mets)
    join_ms = sum(m.kernel_ms["join"] for m in mets)
    join_launches = sum(m.kernel_launches["join"] for m in mets)
    join_evals = sum(m.join_evals for m in mets)
    join_cands = sum(m.join_candidates for m in mets)
    # our kernels per build: init + export, and per iteration indegree,
    # reset, sample, finalize, capacity check, reverse scatter, distances,
    # merge (the two CUB scans per iteration are library kernels, not counted)
    launches = sum(2 + 8 * (len(m.iterations) - 1) for m in mets)
    kernel_ms = {kname: sum(m.kernel_ms[kname] for m in mets) for kname in mets[0].kernel_ms}

    # ---- e2e through the host-pointer C-ABI (pinned host data, graph back to
    # host into page-locked result arrays reused across builds, kg.run(out=))
    pinned = torch.empty((n, d), dtype=torch.float32, pin_memory=True)
    pinned.numpy()[:] = data
    host = pinned.numpy()
    out = kg.KnnGraph(torch.empty((n, k), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32),
                      torch.empty((n, k), dtype=torch.float32, pin_memory=True).numpy(),
                      torch.empty((n, k), dtype=torch.uint8, pin_memory=True).numpy())
    hp = kg.RunParams(k=k, max_candidates=cap, termination_delta=cfg.delta, seed=cfg_r.seed,
                      device=local)
    res = kg.run(host, hp, out=out)  # warm
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    e2e_evals = 0
    h2d = d2h = 0
    for _ in range(args.steps):
        res = kg.run(host, hp, out=out)
        e2e_evals += res.metrics.total_dist_evals
        h2d += res.metrics.h2d_bytes
        d2h += res.metrics.d2h_bytes
    e2e_s = time.perf_counter() - t0

    if dist:
        t = torch.tensor([ms, e2e_s], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_s = float(t[0]), float(t[1])
        c = torch.tensor([evals, e2e_evals], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        evals_all, e2e_all = float(c[0]), float(c[1])
    else:
        evals_all, e2e_all = float(evals), float(e2e_evals)

    out = None
    if rank == 0:
        roof = (u8_roofline(mets, n, d, k, ipeak, peak, args.config) if u8
                else join_roofline(mets, n, d, k, peak, args.config))
        roof["share_of_step"] = round(join_ms / ms, 3)

        # matched recall on a node sample vs the reference (same data, same seed)
        sample = np.random.default_rng(1).choice(n, size=min(n, args.recall_sample),
                                                 replace=False).astype(np.uint32)
        ids_gpu = d_ids.cpu().numpy().astype(np.uint32)
        cpu_baseline = None
        ref_ids = None
        if world == 1 and not args.no_cpu_baseline:
            oracle, kind, O = reference_oracle()
            threads = reference_threads()
            rows = min(n, args.reference_sample or REF_SAMPLE_ROWS.get(cfg.name, 20_000))
            # a build over the whole config also scores the reference's recall
            ev, wall, its, ref_ids = reference_step(O, data, cfg_r, rows, threads)
            cpu_baseline = {
                "value": round(ev / wall, 1), "unit": UNIT, "cores": threads,
                "kind": "reference" if kind.startswith("reference") else "port",
                "sample": (f"{threads} concurrent single-threaded knng::run builds (one per host "
                           f"core; the reference is single-threaded by contract, SPEC.md:375), "
                           f"each on {rows} rows of {cfg.name} (same d, k, cap, delta, seed), "
                           f"{its:.1f} iterations each, {wall:.2f} s wall"),
                "build": ("oracle/_ref/libknng_ref_native.so (the reference's CMake Release flags, "
                          "-march=native)" if kind == "reference_native" else
                          "oracle/_ref/libknng_ref.so (-march=x86-64-v3)" if kind == "reference"
                          else "oracle/lib/libknng_oracle.so (C restatement)"),
                "cpu": oracle.cpu_model(),
            }
            meta = os.path.join(ROOT, "profiles", f"reference_full_{cfg.name}.json")
            if os.path.exists(meta):
                mj = json.load(open(meta))
                cpu_baseline["full_config_single_core"] = {
                    "evals_per_s": round(mj["evals_per_s"], 1),
                    "build_time_s": round(mj["total_wall_s"], 2),
                    "iterations": mj["iterations"], "cpu": mj["cpu"],
                    "source": f"profiles/reference_full_{cfg.name}.json (builder container, "
                              "not this host)"}
        rec = reference_recall_sample(data, k, cfg, ids_gpu, sample, ref_ids)
        builds = args.steps * world
        out = {
            "metric": METRIC, "value": round(evals_all / (ms * 1e-3), 1), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.description}", "n": n, "d": d, "k": k,
                       "max_candidates": cap, "delta": cfg.delta, "seed": cfg.seed,
                       "step": "one complete K-NNG build (init + iterations to termination)",
                       "l2": "inputs larger than L2 (data %.1f MB > 126 MB)" % (n * d * 4 / 1e6),
                       "parallelism": "replicas" if world > 1 else "single-gpu"},
            "build_time_ms": round(ms / args.steps, 3),
            "iterations_per_s": round(iters * world / (ms * 1e-3), 2),
            "iterations_per_build": round(iters / args.steps, 2),
            "recall_at_k": rec,
            "e2e": {"value": round(e2e_all / e2e_s, 1), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d / args.steps),
                    "d2h_bytes_per_step": int(d2h / args.steps),
                    "build_time_ms": round(e2e_s * 1e3 / args.steps, 3)},
            "gpu_launches": int(launches),
            "kernel_ms_per_step": {kk: round(v / args.steps, 3) for kk, v in kernel_ms.items()},
            "roofline": roof,
            "cpu_baseline": cpu_baseline,
            "clocks": clk,
            "builds_timed": builds,
        }
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return None
    oracle, kind, O = reference_oracle()
    cfg = datasets.CONFIGS[args.config]
    data = datasets.generate(cfg)
    threads = reference_threads()
    rows = min(cfg.n, args.reference_sample or REF_SAMPLE_ROWS.get(cfg.name, 20_000))
    for _ in range(args.warmup):
        reference_step(O, data, cfg, rows, threads)
    evals = 0
    wall = 0.0
    iters = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ev, w, its, _ = reference_step(O, data, cfg, rows, threads)
        evals += ev
        wall += w
        iters.append(its)
    elapsed = time.perf_counter() - t0
    value = evals / wall
    sample = (f"{threads} concurrent single-threaded knng::run builds per step (one per host "
              f"core; the reference is single-threaded by contract, SPEC.md:375), each on "
              f"{rows} of the {cfg.n} rows of {cfg.name} (same d, k, cap, delta, seed), "
              f"{np.mean(iters):.1f} iterations per build")
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(wall * 1e3 / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.description}", "n": cfg.n, "d": cfg.d,
                   "k": cfg.k, "max_candidates": cfg.cap, "delta": cfg.delta,
                   "rows_per_build": rows, "builds_per_step": threads,
                   "same_config": rows >= cfg.n},
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": threads,
                         "kind": "reference" if kind.startswith("reference") else "port",
                         "sample": sample, "cpu": oracle.cpu_model(),
                         "build": ("-march=native (reference CMake Release flags)"
                                   if kind == "reference_native" else kind)},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": round(elapsed, 2),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C5", choices=sorted(datasets.CONFIGS))
    ap.add_argument("--recall-sample", type=int, default=5000)
    ap.add_argument("--reference-sample", type=int, default=0,
                    help="rows per reference build (default: REF_SAMPLE_ROWS[config])")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU sharded path even on one GPU (testing)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    rank, world, local = dist_env()
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        out = run_ours(args, rank, world, local)
    if out is not None and rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
