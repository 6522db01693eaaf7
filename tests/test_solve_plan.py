"""Host-side planning of the subdomain solve (band.cu solve_plan + the tile placement tables),
run on CPU through the library's debug entry point: which kernel each configuration gets and
that its shared memory fits a B200 CTA (227 KB)."""
import ctypes as C

import pytest

SMEM_MAX = 227 * 1024


def plan(kd_max, clusters):
    from paper_1508_02977_b200 import _lib
    lib = _lib.load()
    f = lib.ffb_debug_solve_plan
    f.restype = C.c_int
    f.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_longlong), C.POINTER(C.c_int)]
    tile, smem, stage = C.c_int(), C.c_longlong(), C.c_int()
    assert f(kd_max, clusters, C.byref(tile), C.byref(smem), C.byref(stage)) == 0, _lib.last_error()
    return tile.value, smem.value, stage.value


# (kd_max, cluster CTAs per chain, kernel: 1 register-tiled, 2 row-group tile ring, 0 row-batch
# ring) for the configurations' line widths: c1 198 on 8-CTA clusters, c2 297 on 4, c3/c4 423
# on 1 (and on 2- or 4-CTA clusters for a multi-GPU shard), c5 810 on 4
@pytest.mark.parametrize("kd,clusters,tiled", [(198, 8, 1), (297, 4, 1), (423, 1, 2), (810, 4, 0),
                                               (96, 8, 1), (96, 1, 1), (27, 1, 1), (320, 4, 2), (423, 2, 2),
                                               (480, 8, 0), (448, 1, 2), (449, 1, 0),
                                               (161, 1, 2)])
def test_plan_kernel_choice(kd, clusters, tiled):
    tile, smem, stage = plan(kd, clusters)
    assert tile == tiled
    assert 0 < smem <= SMEM_MAX
    if tile == 1:
        # a CTA's share of one line at most a fair share plus one tile, and at least a share
        line = kd * (kd + 1) // 2
        assert line / clusters <= stage <= line / clusters + 2 * 1024 + 64


def test_plan_every_width_fits():
    for clusters in (1, 2, 4, 8):
        for kd in range(2, 834, 7):
            tile, smem, _ = plan(kd, clusters)
            assert 0 < smem <= SMEM_MAX, (kd, clusters)


# the widest line whose operand stage fits next to the slots, per cluster size: one switch
# point each, tiled below it and ring above (the stage shrinks with C, so it grows with C)
@pytest.mark.parametrize("clusters,widest", [(1, 160), (2, 224), (4, 318), (8, 416)])
def test_plan_switch_point(clusters, widest):
    assert plan(widest, clusters)[0] == 1
    # above it: the row-group tiles for one CTA per chain and clusters of 2 / 4, else the ring
    assert plan(widest + 1, clusters)[0] == (2 if clusters <= 4 else 0)


def test_plan_ring_override(monkeypatch):
    monkeypatch.setenv("FFB_SOLVE", "ring")
    tile, smem, _ = plan(297, 4)
    assert tile == 0 and 0 < smem <= SMEM_MAX
    assert plan(423, 1)[0] == 0


def test_plan_row_group_tiles_override(monkeypatch):
    monkeypatch.setenv("FFB_SOLVE", "rt")
    for kd in (27, 96, 160, 448):
        tile, smem, _ = plan(kd, 1)
        assert tile == 2 and 0 < smem <= SMEM_MAX
    assert plan(198, 8)[0] == 1  # clusters: the override does not apply
