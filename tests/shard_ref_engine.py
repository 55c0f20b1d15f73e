"""A CPU (numpy) shard engine with the GpuShardEngine interface, for testing
the multi-process protocol of paper_2112_06630_b200/shard.py over gloo.

Test infrastructure only.  It implements the same per-rank duties as the CUDA
shard — owned-range init, partial in-degree, selection over the owned rows'
edges with reverse offers shipped to their owners, local join of owned active
nodes, merges into owned rows, pre-reduced records for remote targets bounded
by the replicated row maxima, merge of received records — with
deterministic, order-independent rules (no random sampling), so a run over P
ranks must equal the single-rank run exactly.
"""
from __future__ import annotations

import numpy as np
import torch


def _keys(dist: np.ndarray, ids: np.ndarray) -> np.ndarray:
    return (dist.astype(np.float32).view(np.uint32).astype(np.int64) << 32) | ids.astype(np.int64)


def _dist(key: np.ndarray) -> np.ndarray:
    return (key >> 32).astype(np.uint32).view(np.float32)


def _ids(key: np.ndarray) -> np.ndarray:
    return (key & 0xFFFFFFFF).astype(np.int64)


class NumpyShardEngine:
    def __init__(self, data: np.ndarray, k: int, cap: int, rank: int, nranks: int):
        self.data = np.ascontiguousarray(data, np.float32)
        self.n, self.d = self.data.shape
        self.k, self.cap = k, cap
        self.rank, self.nranks = rank, nranks
        self.chunk = (self.n + nranks - 1) // nranks
        self.lo = min(self.n, rank * self.chunk)
        self.hi = min(self.n, (rank + 1) * self.chunk)
        rows = self.chunk * nranks
        self.device = torch.device("cpu")
        self.keys = torch.zeros(rows * k, dtype=torch.int64)
        self.flags = torch.zeros(rows, dtype=torch.int32)
        self.maxd = torch.zeros(rows, dtype=torch.float32)
        self.indeg = torch.zeros(self.n, dtype=torch.int32)
        self.sent_records = 0

    # ------------------------------------------------------------ helpers
    def seeds(self, seed, count):
        return np.random.default_rng(seed).integers(0, 2**63, size=count, dtype=np.int64)

    def sync(self):
        pass

    def _d(self, u, v):
        diff = self.data[u] - self.data[v]
        return np.float32((diff.astype(np.float64) ** 2).sum())

    def _row(self, u):
        return self.keys[u * self.k:(u + 1) * self.k].numpy()

    def _set_row(self, u, keys, flags):
        order = np.argsort(keys, kind="stable")
        keys, flags = keys[order], flags[order]
        self.keys[u * self.k:(u + 1) * self.k] = torch.from_numpy(keys)
        self.flags[u] = int(sum(int(f) << i for i, f in enumerate(flags)))
        self.maxd[u] = float(_dist(keys[-1:])[0])

    def _insert(self, t, proposals):
        """k smallest distinct ids of the row plus proposals; present ids keep
        their stored entry (try_insert's dedup); new entries are is_new."""
        row = self._row(t)
        fl = [(int(self.flags[t]) >> i) & 1 for i in range(self.k)]
        present = {int(i): (int(kk), f) for i, kk, f in zip(_ids(row), row, fl)}
        cand = dict(present)
        for pid, pd in proposals:
            if pid == t or pid in cand:
                continue
            cand[pid] = (int(_keys(np.array([pd]), np.array([pid]))[0]), 1)
        best = sorted(cand.values())[: self.k]
        changed = sum(1 for kk, f in best if int(_ids(np.array([kk]))[0]) not in present)
        self._set_row(t, np.array([b[0] for b in best], np.int64),
                      np.array([b[1] for b in best], np.int64))
        return changed

    # ------------------------------------------------------------ protocol
    def init(self, seed):
        for u in range(self.lo, self.hi):
            rng = np.random.default_rng([int(seed) & 0x7FFFFFFF, u])
            pool = np.delete(np.arange(self.n), u)
            ids = rng.choice(pool, size=self.k, replace=False)
            dists = np.array([self._d(u, v) for v in ids], np.float32)
            self._set_row(u, _keys(dists, ids), np.ones(self.k, np.int64))

    def _owned_ids(self):
        k = self.k
        keys = self.keys[self.lo * k:self.hi * k].numpy().reshape(-1, k)
        return _ids(keys)

    def degree(self):
        """Partial in-degree of the owned rows' edges (the runner sums them)."""
        self.indeg.zero_()
        ids = self._owned_ids()
        if ids.size:
            self.indeg += torch.from_numpy(
                np.bincount(ids.reshape(-1), minlength=self.n).astype(np.int32))
        return self.indeg

    def sample(self, seed):
        """Owned rows' edges only: reverse edges (u -> v) to owned v stay
        local, the others become offers {v, u, flag, 0} for owner(v)."""
        ids = self._owned_ids()
        flags = self.flags[self.lo:self.hi].numpy()
        self._rev = {t: [] for t in range(self.lo, self.hi)}
        out = [[] for _ in range(self.nranks)]
        for r, u in enumerate(range(self.lo, self.hi)):
            for i in range(self.k):
                v, f = int(ids[r, i]), (int(flags[r]) >> i) & 1
                if self.lo <= v < self.hi:
                    self._rev[v].append((u, f))
                else:
                    out[min(self.nranks - 1, v // self.chunk)].append((v, u, f, 0))
        counts = [len(o) for o in out]
        segs = [torch.from_numpy(np.array(o, np.int64).reshape(-1).astype(np.int32))
                for o in out]
        self.seg_cap = max(counts + [1])
        return counts, segs

    def offers(self, recv):
        rec = recv.numpy().reshape(-1, 4)
        for v, u, f, _ in rec:
            self._rev[int(v)].append((int(u), int(f)))

    def step(self):
        n, k, cap = self.n, self.k, self.cap
        ids = self._owned_ids()
        flags = self.flags[self.lo:self.hi].numpy()
        maxd0 = self.maxd[:n].numpy().copy()
        # lists of the owned nodes: forward entries, then reverse edges in
        # source order, first occurrence wins, each list the cap smallest ids
        lists = {}
        for r, t in enumerate(range(self.lo, self.hi)):
            seen = {}
            for i in range(k):
                seen.setdefault(int(ids[r, i]), int((flags[r] >> i) & 1))
            for x, f in sorted(self._rev[t]):
                seen.setdefault(int(x), int(f))
            new = sorted(x for x, f in seen.items() if f)[:cap]
            old = sorted(x for x, f in seen.items() if not f)[:cap]
            lists[t] = (new, old)
        # flag_consumed on owned rows
        for r, (t, (new, _)) in enumerate(lists.items()):
            fl = int(self.flags[t])
            for i in range(k):
                if int(ids[r, i]) in new:
                    fl &= ~(1 << i)
            self.flags[t] = fl
        # local join of owned active nodes
        props = {}
        evals = cands = 0
        for u, (new, old) in lists.items():
            if not new:
                continue
            evals += len(new) * (len(new) - 1) // 2 + len(new) * len(old)
            cands += len(new) + len(old)
            pairs = [(new[a], new[b]) for a in range(len(new)) for b in range(a + 1, len(new))]
            pairs += [(x, y) for x in new for y in old]
            for x, y in pairs:
                dd = self._d(x, y)
                props.setdefault(x, []).append((y, dd))
                props.setdefault(y, []).append((x, dd))
        changes = 0
        records = []
        for t, plist in sorted(props.items()):
            if self.lo <= t < self.hi:
                changes += self._insert(t, plist)
            else:
                # pre-reduced export: the k best distinct
                # proposals below t's (replicated) row maximum
                entered = {}
                for pid, pd in plist:
                    if pd >= maxd0[t] or pid == t or pid in entered:
                        continue
                    entered[pid] = pd
                for d_, pid in sorted((d_, i) for i, d_ in entered.items())[:k]:
                    records.append((t, pid, int(np.float32(d_).view(np.uint32))))
        self._local_changes = changes
        owner = [min(self.nranks - 1, t // self.chunk) for t, _, _ in records]
        order = np.argsort(owner, kind="stable") if records else []
        recs = [records[i] for i in order]
        counts = [0] * self.nranks
        for i in order:
            counts[owner[i]] += 1
        flat = np.array(recs, np.int64).reshape(-1) if recs else np.zeros(0, np.int64)
        send = torch.from_numpy(flat.astype(np.uint32).view(np.int32).copy())
        return dict(evals=evals, cands=cands, active=len(lists), send_counts=counts, send=send)

    def merge(self, recv):
        rec = recv.numpy().view(np.uint32).reshape(-1, 3)
        by_t = {}
        for t, pid, bits in rec:
            by_t.setdefault(int(t), []).append((int(pid), np.uint32(bits).view(np.float32)))
        changes = self._local_changes
        for t, plist in sorted(by_t.items()):
            changes += self._insert(t, plist)
        return changes

    def export(self):
        rows = self.keys[self.lo * self.k:self.hi * self.k].numpy().reshape(-1, self.k)
        return (torch.from_numpy(_ids(rows).astype(np.int32)),
                torch.from_numpy(_dist(rows).copy()))
