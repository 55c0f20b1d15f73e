"""GPU parity of the byte-valued join (csrc/join_u8.cu).

Data whose coordinates are all integers in [0, 255] (C2's pixels) takes the
integer tensor-core path automatically; its lane sums are exact integers, so
every distance must be bit-identical to the FP32 tile kernel's (forced with
KNNG_JOIN_U8=0) and to the reference (the C2 cases of test_gpu_parity.py run
through this path by default).
"""
import numpy as np
import pytest

import paper_2112_06630_b200 as kg

from test_gpu_parity import compare_step, make_data

pytestmark = pytest.mark.gpu


def u8_data(n, d, seed, sparse=True):
    rng = np.random.default_rng(seed)
    x = rng.integers(0, 256, size=(n, d)).astype(np.float32)
    if sparse:
        x[rng.random((n, d)) < 0.7] = 0.0
    return x


@pytest.mark.parametrize("kind,n,k,cap,seed,t", [
    ("C2", 3000, 20, 50, 1, 1), ("C2", 3000, 20, 50, 1, 2), ("C2", 3000, 20, 50, 1, 6),
    ("U8_100", 2000, 12, 20, 3, 1), ("U8_128", 3000, 10, 50, 4, 2), ("U8_24", 1500, 8, 15, 5, 1),
    ("U8_1000", 1500, 10, 40, 6, 1), ("U8_1000", 1500, 10, 40, 6, 3),
])
def test_u8_step_equals_fp32_kernel_and_oracle(gpu, restated, monkeypatch, kind, n, k, cap, seed,
                                               t):
    data = make_data(kind, n, seed) if kind == "C2" else u8_data(n, int(kind[3:]), seed)
    gi, c, go, _, ev_ref = restated.capture_step(data, k, cap, seed, t)
    cands = kg.CandidateSet(c.ids, c.new_counts, c.old_counts)
    out = {}
    for mode in ("0", "1", "noswap", "mixed", "staged", "tc"):
        # "1": the default (warp-per-node kernel); "mixed": nodes with more
        # than 16 new candidates through the opt-in staged kernel (CTA per
        # node, rows in shared memory) where it fits, the rest through the
        # warp-per-node kernel; "staged": every node through the staged kernel
        monkeypatch.setenv("KNNG_JOIN_U8", "0" if mode == "0" else "1")
        monkeypatch.setenv("KNNG_U8_STAGED", "1" if mode in ("mixed", "staged") else "0")
        monkeypatch.setenv("KNNG_U8_HEAVY", "0" if mode == "staged" else "16")
        # "noswap": nodes with nn <= 8 keep the 16 (new) x 8 tile shape
        monkeypatch.setenv("KNNG_U8_SWAP", "0" if mode == "noswap" else "1")
        # "tc": the tcgen05 kernel (join_u8_tc.cu) where its shapes are
        # supported (Kl = 128: C2, U8_1000), the warp kernel otherwise
        monkeypatch.setenv("KNNG_U8_TC", "1" if mode == "tc" else "0")
        out[mode] = kg.compute_step(data, gi.ids, gi.dists, gi.flags, cands)
    g8 = out["1"][0]
    assert out["1"][3] == ev_ref
    for mode in ("noswap", "mixed", "staged", "tc"):
        assert out[mode][3] == ev_ref
        st3 = compare_step(gi, out[mode][0], g8)
        assert st3["mismatch"] == 0 and st3["bit_exact"] == st3["common"], (mode, st3)
    st = compare_step(gi, go, g8, restated=restated, data=data)
    assert st["mismatch"] == 0 and st["flag_mismatch"] == 0, st
    # byte-valued data: fused and unfused paths agree, so every stored
    # distance is the reference's own value
    assert st["bit_exact"] == st["common"], st
    st2 = compare_step(gi, out["0"][0], g8)
    assert st2["mismatch"] == 0 and st2["bit_exact"] == st2["common"], st2


@pytest.mark.parametrize("d", [784, 100, 24])
def test_u8_candidate_distances_bit_exact(gpu, restated, d):
    """Every (new, candidate) distance of a step, unfiltered, against the
    reference's mutual_block_distances / block_l2_sq values."""
    data = u8_data(1200, d, 7)
    gi, c, _, _, _ = restated.capture_step(data, 10, 20, 7, 1)
    cands = kg.CandidateSet(c.ids, c.new_counts, c.old_counts)
    got = kg.candidate_distances(data, cands)
    n = data.shape[0]
    stride = (d + 7) // 8 * 8
    pdata = np.zeros((n, stride), np.float32)  # the reference's padded rows
    pdata[:, :d] = data
    for u in range(0, n, 37):
        nn, no = int(c.new_counts[u]), int(c.old_counts[u])
        if nn == 0:
            continue
        ids = np.concatenate([c.ids[u, :nn], c.ids[u, 20:20 + no]])
        for i in range(nn):
            for j in range(nn + no):
                if j < nn and j <= i:
                    continue
                ref = restated.l2_sq(pdata[ids[i]], pdata[ids[j]])
                assert np.float32(got[u][i, j]).view(np.uint32) == np.float32(ref).view(np.uint32)


def test_u8_build_matches_fp32_build(gpu, monkeypatch):
    data = make_data("C2", 4000)
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("KNNG_JOIN_U8", mode)
        res[mode] = kg.run(data, kg.RunParams(k=20, max_candidates=50, seed=0))
    ex, _ = kg.brute_force_knng(data, 20)
    r0, r1 = kg.recall(res["0"].graph.ids, ex), kg.recall(res["1"].graph.ids, ex)
    assert abs(r0 - r1) <= 0.005, (r0, r1)


@pytest.mark.parametrize("kind,d", [("C2", 784), ("U8", 100), ("U8", 24)])
def test_u8_init_distances_bit_exact(gpu, restated, kind, d):
    """init_random's distances from the integer lane sums equal the reference's
    scalar l2_sq on the padded rows (graph.hpp:60), bit for bit."""
    data = make_data("C2", 1500) if kind == "C2" else u8_data(1500, d, 9)
    g, _, ev = kg.init_random(data, 10, 5)
    n = data.shape[0]
    stride = (data.shape[1] + 7) // 8 * 8
    pdata = np.zeros((n, stride), np.float32)
    pdata[:, :data.shape[1]] = data
    for u in range(0, n, 29):
        for i in range(10):
            want = restated.l2_sq(pdata[u], pdata[g.ids[u, i]])
            assert np.float32(g.dists[u, i]).view(np.uint32) == np.float32(want).view(np.uint32)
