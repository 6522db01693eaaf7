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


def test_run_pipeline_files_end_to_end(ctx, tmp_path):
    """pipeline.cpp:110-120: PGM frames in, .flo + metrics CSV out; the metrics equal
    compute_metrics of the returned flow against the written truth."""
    from paper_1508_02977_b200 import synth
    f0, f1, flow, cfg = synth.make("c1")
    ff.save_pgm(str(tmp_path / "f0.pgm"), f0 / 255.0)
    ff.save_pgm(str(tmp_path / "f1.pgm"), f1 / 255.0)
    ff.write_flo(str(tmp_path / "gt.flo"), ff.FloField(flow[0].astype(np.float32),
                                                       flow[1].astype(np.float32)))
    pc = ff.PipelineConfig(str(tmp_path / "f0.pgm"), str(tmp_path / "f1.pgm"),
                           str(tmp_path / "gt.flo"), str(tmp_path / "out.flo"),
                           str(tmp_path / "m.csv"),
                           ff.RunConfig(sigma=cfg.sigma, parts=cfg.parts, overlap=cfg.overlap,
                                        adapt_iters=cfg.n_passes), scale_255=True)
    r = ff.run_pipeline(pc, ctx=ctx)
    out = ff.read_flo(str(tmp_path / "out.flo"))
    assert np.array_equal(out.u, r.result.flow.u1.astype(np.float32))
    m = ff.compute_metrics(r.result.flow, ff.read_flo(str(tmp_path / "gt.flo")), ctx=ctx)
    assert (m.aae_deg, m.ee, m.valid) == (r.metrics.aae_deg, r.metrics.ee, r.metrics.valid)
    assert r.metrics.valid == f0.size and r.metrics.ee < 1.0  # the rotation is recovered
    lines = (tmp_path / "m.csv").read_text().splitlines()
    assert lines[0] == "mode,aae_deg,ee,valid_pixels" and lines[1].startswith("illum_on,")
