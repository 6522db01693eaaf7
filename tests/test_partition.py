"""Host-side decomposition (schwarz.cpp:16-128) against the reference, bit for bit, and
the reference's own known answers (test_schwarz.cpp:46-147, acceptance.cpp:246-263)."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1508_02977_b200 import flowfem as ff


def test_split_ratio_known_answers():
    # test_schwarz.cpp:46-68: 4 parts of a 96x80 image etc.
    s = ff.enumerate_splits(96, 80, 4)
    assert [(x.parts_x, x.parts_y) for x in s] == [(1, 4), (2, 2), (4, 1)]
    c = ff.choose_split(96, 80, 4)
    assert (c.parts_x, c.parts_y) == (2, 2)
    assert abs(c.ratio - (48 * 40) / (2 * (48 + 40))) < 1e-12
    # ties prefer parts_x >= parts_y (square image)
    c = ff.choose_split(64, 64, 2)
    assert (c.parts_x, c.parts_y) == (2, 1)
    # acceptance.cpp criterion 5: 12 parts on 4:3 -> 4x3
    c = ff.choose_split(640, 480, 12)
    assert (c.parts_x, c.parts_y) == (4, 3)


def test_split_matches_reference(ref):
    rng = np.random.default_rng(3)
    for _ in range(200):
        W, H, n = int(rng.integers(2, 3000)), int(rng.integers(2, 3000)), int(rng.integers(1, 300))
        c = ff.choose_split(W, H, n)
        assert (c.parts_x, c.parts_y, c.ratio) == ref.choose_split(W, H, n)


def test_configured_splits_and_partitions_golden():
    g = json.load(open(os.path.join(GOLDEN, "partitions.json")))
    for name, (px, py, ratio) in g["splits"].items():
        from paper_1508_02977_b200 import synth
        cfg = synth.CONFIGS[name]
        c = ff.choose_split(cfg.W, cfg.H, cfg.parts)
        assert (c.parts_x, c.parts_y) == (px, py)
        assert c.ratio == ratio
    for key, p in g["partitions"].items():
        flat = ff.build_partition_flat(p["W"], p["H"], p["px"], p["py"], p["ov"])
        assert flat.size == p["length"], key
        assert hashlib.sha256(flat.astype("<i4").tobytes()).hexdigest() == p["sha256"], key


@pytest.mark.parametrize("W,H,px,py,ov", [(20, 17, 2, 2, 3), (96, 80, 2, 2, 5), (31, 29, 3, 2, 2),
                                          (64, 64, 1, 1, 0), (50, 40, 4, 1, 2), (13, 11, 1, 2, 1),
                                          (128, 128, 2, 2, 4), (300, 200, 5, 4, 7)])
def test_partition_bit_exact(ref, port, W, H, px, py, ov):
    mine = ff.build_partition_flat(W, H, px, py, ov)
    assert np.array_equal(mine, ref.build_partition(W, H, px, py, ov))
    assert np.array_equal(mine, port.build_partition(W, H, px, py, ov))


def test_partition_invariants():
    # test_schwarz.cpp:86-140: cores tile the image; ext = core +- ov clipped; gamma grouped
    W, H, px, py, ov = 97, 83, 3, 4, 4
    P = ff.build_partition(W, H, px, py, ov)
    cover = np.zeros((H, W), int)
    for s in P.parts:
        cover[s.core.y0:s.core.y1, s.core.x0:s.core.x1] += 1
        assert s.ext.x0 == max(0, s.core.x0 - ov) and s.ext.x1 == min(W, s.core.x1 + ov)
        assert s.boundary == sorted(s.boundary)
        allg = sorted(v for nb in s.neighbors for v in nb.gamma)
        assert allg == s.boundary
        for nb in s.neighbors:
            q = P.parts[nb.part]
            for v in nb.gamma:
                assert q.core.contains(v % W, v // W)
    assert (cover == 1).all()


def test_partition_rejects():
    with pytest.raises(ff.FlowfemError, match="schwarz.build_partition: core 10x20 not larger "
                                              "than twice the overlap 5"):
        ff.build_partition(20, 20, 2, 1, 5)
    with pytest.raises(ff.FlowfemError, match="overlap must be >= 1"):
        ff.build_partition(20, 20, 2, 1, 0)
    with pytest.raises(ff.FlowfemError, match="part counts must be >= 1"):
        ff.build_partition(20, 20, 0, 1, 1)
    with pytest.raises(ff.FlowfemError, match="n_parts must be >= 1"):
        ff.enumerate_splits(20, 20, 0)


def test_assign_workers_round_robin():
    # test_schwarz.cpp:80-84
    assert ff.assign_workers(7, 3) == [0, 1, 2, 0, 1, 2, 0]
    with pytest.raises(ff.FlowfemError, match="counts must be >= 1"):
        ff.assign_workers(0, 3)
