"""Repro of the sharded hub-path bug: a 2-rank in-process split
of C2-shaped data.  Run with KNNG_SHARD_U8=0 (fails every time) and a
KNNG_JOIN_CHECKS=1 build (KNNG_CUDA_LIB=scripts/libknng_cuda_chk.so)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2112_06630_b200 as kg
from paper_2112_06630_b200 import datasets
from paper_2112_06630_b200.shard import GpuShardEngine, seed_sequence

def split(kind):
  cfg = datasets.CONFIGS[kind]
  data = datasets.generate(cfg)[:12000]
  n, k = data.shape[0], cfg.k
  params = kg.RunParams(k=k, max_candidates=cfg.cap, seed=0)
  dd = torch.from_numpy(data).cuda()
  engs = [GpuShardEngine(dd, params, r, 2) for r in range(2)]
  seeds = seed_sequence(0, 31)
  for e in engs:
      e.init(int(seeds[0]))
  chunk = engs[0].chunk


  def allgather():
      for buf, w in (("keys", k), ("flags", 1), ("maxd", 1)):
          for r in range(2):
              src = getattr(engs[r], buf)[r * chunk * w:(r + 1) * chunk * w]
              getattr(engs[1 - r], buf)[r * chunk * w:(r + 1) * chunk * w].copy_(src)
      torch.cuda.synchronize()


  allgather()
  for it in range(1, 31):
      steps = []
      for r, e in enumerate(engs):
          print("step", it, "rank", r, flush=True)
          steps.append(e.step(int(seeds[it])))
      ch = 0
      for r in range(2):
          print("merge", it, "rank", r, "records", steps[1 - r]["send"].numel() // 3, flush=True)
          ch += engs[r].merge(steps[1 - r]["send"].clone())
      allgather()
      print("iteration", it, "changes", ch, flush=True)
      if ch < params.termination_delta * n * k:
          break


for kind in [a for a in sys.argv[1:] if not a.startswith("--")] or ["C2"]:
    print("split", kind, flush=True)
    split(kind)
    if "--run" in sys.argv:  # what the pytest case does after its split
        d = datasets.generate(datasets.CONFIGS[kind])[:12000]
        kg.brute_force_knng(d, datasets.CONFIGS[kind].k)
        kg.run(d, kg.RunParams(k=datasets.CONFIGS[kind].k,
                               max_candidates=datasets.CONFIGS[kind].cap, seed=0))
        print("single-GPU run done", flush=True)
print("done")
