"""Per-phase host timing of the sharded loop at world size 1 (diagnostics)."""
import os, sys, time, socket
sys.path.insert(0, ".")
import numpy as np, torch, torch.distributed as dist
import paper_2112_06630_b200 as kg
from paper_2112_06630_b200 import datasets
from paper_2112_06630_b200.shard import GpuShardEngine, _allgather_rows
torch.cuda.set_device(0)
if "RANK" in os.environ:  # under torchrun, like bench.py
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
else:
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
cfg = datasets.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
data = datasets.generate(cfg)
params = kg.RunParams(k=cfg.k, max_candidates=cfg.cap, seed=0)
eng = GpuShardEngine(torch.from_numpy(data).cuda(), params, 0, 1)
seeds = eng.seeds(0, 32)
for rep in range(2):
    eng.init(int(seeds[0])); _allgather_rows(eng); torch.cuda.synchronize()
    acc = {}
    def tick(name, t0):
        torch.cuda.synchronize(); t1 = time.perf_counter(); acc[name] = acc.get(name, 0) + t1 - t0; return t1
    for it in range(1, 17):
        t = time.perf_counter()
        st = eng.step(int(seeds[it])); t = tick("step", t)
        sc = torch.tensor([3 * c for c in st["send_counts"]], dtype=torch.int64, device="cuda")
        rcnt = torch.empty_like(sc); dist.all_to_all_single(rcnt, sc); rc = rcnt.tolist(); t = tick("a2a_counts", t)
        recv = torch.empty(int(sum(rc)), dtype=torch.int32, device="cuda")
        dist.all_to_all_single(recv, st["send"], output_split_sizes=rc, input_split_sizes=sc.tolist()); t = tick("a2a_recs", t)
        ch = eng.merge(recv); t = tick("merge", t)
        _allgather_rows(eng); t = tick("allgather", t)
        tot = torch.tensor([ch, st["evals"], st["cands"]], dtype=torch.float64, device="cuda")
        dist.all_reduce(tot); v = tot.tolist(); t = tick("allreduce", t)
    print({k: round(v * 1e3, 2) for k, v in acc.items()}, flush=True)
from paper_2112_06630_b200.shard import run_sharded
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    res = run_sharded(eng, params)
    torch.cuda.synchronize(); print("run_sharded ms", round((time.perf_counter() - t) * 1e3, 2),
          "iters", len(res.metrics.iterations) - 1,
          "per-iter wall ms", [round(i.wall_time_s * 1e3, 2) for i in res.metrics.iterations], flush=True)
eng.close()
dist.destroy_process_group()
