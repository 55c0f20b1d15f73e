"""Host-side evaluation helpers of the Python mirror, restating the
reference's own unit tests (no GPU): scaling_exponent (oracle.hpp:147-171;
test_oracle.cpp:138-154) and window_cluster_fraction (reorder.hpp:61-86;
test_reorder.cpp:85-123)."""
import numpy as np
import pytest

import paper_2112_06630_b200 as kg


def test_scaling_exponent_known_answers():
    sizes = [1000, 2000, 4000, 8000]
    assert kg.scaling_exponent(sizes, [3.0 * s for s in sizes]) == pytest.approx(1.0, rel=1e-9)
    assert kg.scaling_exponent(sizes, [0.5 * s * s for s in sizes]) == pytest.approx(2.0, rel=1e-9)
    with pytest.raises(kg.InvalidArgument):
        kg.scaling_exponent([10, 20], [10, 20])
    with pytest.raises(kg.InvalidArgument):
        kg.scaling_exponent([10, 30, 20], [1, 2, 3])
    with pytest.raises(kg.InvalidArgument):
        kg.scaling_exponent([10, 20, 30], [1, 0, 3])


def test_window_fractions_identity_on_contiguous_clusters():
    # clusters laid out contiguously, identity permutation: aligned windows pure
    n, window, c = 8000, 1000, 8
    labels = np.repeat(np.arange(c), n // c)
    rows = kg.window_cluster_fraction(labels, np.arange(n), window)
    for start, cl, f in rows:
        if start % window == 0:
            assert f == (1.0 if cl == start // window else 0.0)


def test_window_fractions_flat_for_random_permutation():
    n, c = 16384, 8
    labels = np.arange(n) % c
    sigma = np.random.default_rng(3).permutation(n)
    rows = kg.window_cluster_fraction(labels, sigma, 2000)
    assert all(abs(f - 0.125) < 0.04 for _, _, f in rows)


def test_window_fractions_walk_and_sums():
    n, window = 4096, 512
    labels = np.random.default_rng(9).integers(0, 8, n)
    rows = kg.window_cluster_fraction(labels, np.random.default_rng(1).permutation(n), window)
    starts = sorted({r[0] for r in rows})
    # starts advance by window / 4; the last start is n - window
    assert starts[:3] == [0, 128, 256] and starts[-1] == n - window
    sums = {}
    for s, _, f in rows:
        sums[s] = sums.get(s, 0.0) + f
    assert len(sums) > 1 and all(abs(v - 1.0) < 1e-12 for v in sums.values())
    with pytest.raises(kg.InvalidArgument):
        kg.window_cluster_fraction(labels[:-1], np.arange(n), window)
    with pytest.raises(kg.InvalidArgument):
        kg.window_cluster_fraction(labels, np.arange(n), n + 1)
