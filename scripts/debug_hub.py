import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2112_06630_b200 as kg
import oracle
if not oracle.available("restated"):
    oracle.build("restated")
restated = oracle.load("restated")
n, d, k, cap, hub = 2400, 32, 10, 12, 7
rng = np.random.default_rng(21)
data = rng.standard_normal((n, d), dtype=np.float32)
data[hub] = data.mean(axis=0)
g0, _ = restated.init_random(data, k, 5)
ids = np.zeros((n, 2 * cap), np.uint32); nc = np.zeros(n, np.uint32); oc = np.zeros(n, np.uint32)
for u in range(n):
    pool = rng.choice(np.delete(np.arange(n), [u, hub]), size=cap - 1 + 4, replace=False)
    new = [hub] + pool[: cap - 1].tolist() if u != hub else pool[:cap].tolist()
    ids[u, : len(new)] = new; nc[u] = len(new)
    old = pool[cap - 1:cap + 3].tolist(); ids[u, cap: cap + len(old)] = old; oc[u] = len(old)
go, ch_ref, ev_ref = restated.compute_step(data, g0, oracle.Cands(ids, nc, oc))
g, rev, ch, ev = kg.compute_step(data, g0.ids, g0.dists, g0.flags, kg.CandidateSet(ids, nc, oc))
for u in range(n):
    ref = dict(zip(go.ids[u].tolist(), go.dists[u].tolist()))
    gpu = dict(zip(g.ids[u].tolist(), g.dists[u].tolist()))
    if set(ref) != set(gpu):
        print("row", u, "hub" if u == hub else "")
        print(" ref-only", {v: ref[v] for v in set(ref) - set(gpu)})
        print(" gpu-only", {v: gpu[v] for v in set(gpu) - set(ref)})
        print(" ref max", max(ref.values()), "gpu max", max(gpu.values()))
        print(" init", sorted(zip(g0.dists[u].tolist(), g0.ids[u].tolist()))[:3])
t = 1663
for u in range(n):
    lst = ids[u, :nc[u]].tolist() + ids[u, cap:cap + oc[u]].tolist()
    if lst.count(t) > 1 or (t in lst and len(set(lst)) != len(lst)):
        print("dup list", u, lst)
    if u == t and t in lst:
        print("self in own list")
rows_with_t = [u for u in range(n) if t in ids[u, :nc[u]].tolist() + ids[u, cap:cap + oc[u]].tolist()]
print("lists naming t:", len(rows_with_t), rows_with_t[:20])
print("nc/oc of those", [(int(nc[u]), int(oc[u])) for u in rows_with_t[:20]])
dup = [u for u in range(n) if len(set(ids[u, :nc[u]].tolist() + ids[u, cap:cap + oc[u]].tolist())) != nc[u] + oc[u]]
print("lists with duplicates:", len(dup), dup[:5])
