"""Tile geometry of the 5 x 10 tile join (csrc/join5_geom.cuh), checked on the
host through knng_cuda_debug_join5_pairs (no GPU): for every list shape the
build supports, the tiles evaluate each pair of compute_step (reference
descent.hpp:82-153: new x new once, new x old once, never old x old) exactly
once, and in the reference's arithmetic class -- fused inside full 5 x 5 /
triangular blocks (block_core / tri_core5, distance.hpp:134-190), unfused
wherever a leftover (index >= the last multiple of 5) candidate is involved."""
import ctypes

import numpy as np
import pytest

from paper_2112_06630_b200 import _native


def tile_pairs(nn, no, thin):
    lib = ctypes.CDLL(_native.LIB_PATH)
    fn = lib.knng_cuda_debug_join5_pairs
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, ctypes.c_void_p,
                   ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32)]
    cap = (nn + no) * (nn + no) + 64
    out = np.zeros((cap, 3), np.uint32)
    count = ctypes.c_uint32(0)
    tiles = fn(nn, no, int(thin), out.ctypes.data, cap, ctypes.byref(count))
    assert count.value <= cap
    return tiles, out[: count.value]


def expected_pairs(nn, no):
    """{(lo, hi): fused} over candidate positions (new 0..nn-1, old nn..nn+no-1)."""
    fn, fo = nn - nn % 5, no - no % 5
    exp = {}
    for i in range(nn):
        for j in range(i + 1, nn):
            exp[(i, j)] = i < fn and j < fn
        for j in range(no):
            exp[(i, nn + j)] = i < fn and j < fo
    return exp


SHAPES = [(nn, no) for nn in range(0, 65) for no in range(0, 65)]


@pytest.mark.parametrize("thin", [False, True])
def test_every_pair_once_in_its_class(thin):
    for nn, no in SHAPES:
        tiles, got = tile_pairs(nn, no, thin)
        exp = expected_pairs(nn, no)
        seen = {}
        for r, c, fused in got.tolist():
            key = (min(r, c), max(r, c))
            assert key not in seen, (nn, no, thin, key)
            seen[key] = bool(fused)
        assert seen == exp, (nn, no, thin, len(seen), len(exp))
        if nn == 0:
            assert tiles == 0


def test_tile_counts_against_the_cost_model():
    """Tile counts the measurements in profiles/README.md rest on."""
    # nn = 7, no = 23: 3 fused + 3 leftover-row tiles (ten 8 x 8 tiles before)
    assert tile_pairs(7, 23, False)[0] == 6
    # a late node, one new and 23 old candidates: one thin tile, or three 5 x 10
    assert tile_pairs(1, 23, True)[0] == 1
    assert tile_pairs(1, 23, False)[0] == 3
    # all-new iteration-1 node of C5: 20 fused tiles, no leftovers
    assert tile_pairs(40, 0, True)[0] == 20
    # thin tiles only when at most two leftover rows are live
    assert tile_pairs(13, 0, True)[0] == tile_pairs(13, 0, False)[0]
