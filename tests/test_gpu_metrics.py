"""compute_metrics (metrics.cpp:75-100) as a device reduction against the reference's."""
import numpy as np
import pytest

from paper_1508_02977_b200 import flowfem as ff

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("H,W", [(37, 53), (388, 584)])
def test_metrics_match_reference(ctx, ref, H, W):
    import pyoracle as po
    rng = np.random.default_rng(H)
    flow = rng.normal(0, 2, (3, H, W))
    tu = (flow[0] + rng.normal(0, 0.3, (H, W))).astype(np.float32)
    tv = (flow[1] + rng.normal(0, 0.3, (H, W))).astype(np.float32)
    tu[0, :5] = 1e10
    tv[1, 3] = np.nan
    tu[2, 2] = -np.inf
    a, e, k = po.ref_compute_metrics(flow, tu, tv)
    m = ff.compute_metrics(ff.FlowState.from_planes(flow), ff.FloField(tu, tv), ctx=ctx)
    assert m.valid == k == H * W - 7
    assert abs(m.aae_deg - a) <= 1e-12 * a
    assert abs(m.ee - e) <= 1e-12 * e


def test_metrics_no_valid_and_size_mismatch(ctx):
    flow = ff.FlowState.from_planes(np.zeros((3, 4, 5)))
    bad = np.full((4, 5), 2e9, np.float32)
    m = ff.compute_metrics(flow, ff.FloField(bad, bad), ctx=ctx)
    assert (m.aae_deg, m.ee, m.valid) == (0.0, 0.0, 0)
    with pytest.raises(ff.FlowfemError, match="metrics.compute_metrics: flow and ground truth sizes differ"):
        ff.compute_metrics(flow, ff.FloField(np.zeros((5, 4), np.float32), np.zeros((5, 4), np.float32)), ctx=ctx)
