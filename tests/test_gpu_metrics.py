"""Metrics on the GPU (paper_2101_10994_b200.metrics) vs the reference's
golden fixtures (tests/golden/make_golden_metrics.py) on the planted LOD4
torus. Bars follow BASELINE.json: hit masks >= 99.9 % equal, depth within
2e-3, SDF values within 1e-4; exact where the arithmetic is the same
(nearest-neighbour distances, cameras)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HIT_AGREE = 0.999
DEPTH_TOL = 2e-3
SDF_TOL = 1e-4


@pytest.fixture(scope="module")
def env(golden):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2101_10994_b200 as ng
    from paper_2101_10994_b200 import metrics as M
    from paper_2101_10994_b200 import scenes
    tor = scenes.Torus(0.5, 0.2)
    svo = ng.build_octree(tor, 4, golden("octree")["samples_b"])
    fld = scenes.planted_field(svo, tor, seed=0, device_sdf=False)
    return ng, M, tor, fld, golden("metrics")


def _rays(ng, g):
    return ng.RayBundle(g["rays_o"], g["rays_d"])


def _agree(a, b):
    return float(np.mean(np.asarray(a) == np.asarray(b)))


def test_trace_oracle_rays(env):
    ng, M, tor, fld, g = env
    hit, t = M.trace_oracle_rays(tor, _rays(ng, g))
    assert _agree(hit, g["oracle_hit"]) >= HIT_AGREE
    both = hit & g["oracle_hit"]
    assert both.sum() > 100
    assert np.max(np.abs(t[both] - g["oracle_t"][both])) <= DEPTH_TOL
    # a host-callable oracle (no device SDF) follows the same rules
    hit2, t2 = M.trace_oracle_rays(lambda p: tor(p), _rays(ng, g))
    assert _agree(hit2, g["oracle_hit"]) >= HIT_AGREE


def test_trace_field_rays(env):
    ng, M, tor, fld, g = env
    hit, t = M.trace_field_rays(fld, _rays(ng, g), 4.0)
    assert _agree(hit, g["field_hit"]) >= HIT_AGREE
    both = hit & g["field_hit"]
    assert np.max(np.abs(t[both] - g["field_t"][both])) <= DEPTH_TOL


def test_sample_predicted_surface(env):
    ng, M, tor, fld, g = env
    pts = M.sample_predicted_surface(fld, 500, rng_seed=2, lod=4.0)
    assert pts.shape == (500, 3)
    d = M.PointGrid(g["surf_pts"]).nearest_dist(pts)
    assert np.mean(d <= DEPTH_TOL) >= 0.99
    assert np.all(np.abs(fld.predict(pts, 4)) <= ng.RenderConfig().delta + SDF_TOL)
    np.testing.assert_array_equal(pts, M.sample_predicted_surface(fld, 500, rng_seed=2, lod=4.0))
    assert M.sample_predicted_surface(fld, 0).shape == (0, 3)


def test_signed_extension_and_giou(env):
    ng, M, tor, fld, g = env
    for lv in (4, 2):
        v = M.predict_signed_extension(fld, g["ext_pts"], lv)
        np.testing.assert_allclose(v, g[f"ext_l{lv}"], atol=SDF_TOL, rtol=0)
    gi = M.giou(fld, tor, 4096, rng_seed=4, level=4)
    assert gi == pytest.approx(float(g["giou"]), abs=0.5)
    assert M.giou(fld, tor, 2048, rng_seed=1, level=4) > 80.0
    with pytest.raises(ng.ConfigError):
        M.giou(fld, tor, 0)


def test_nearest_neighbours_and_chamfer_exact(env):
    ng, M, tor, fld, g = env
    np.testing.assert_array_equal(M.PointGrid(g["truth_pts"]).nearest_dist(g["nn_q"]), g["nn_d"])
    assert M.chamfer_l1(g["surf_pts"], g["truth_pts"]) == float(g["chamfer"])
    assert M.chamfer_l1(g["truth_pts"], g["truth_pts"]) == 0.0
    with pytest.raises(ng.ConfigError):
        M.chamfer_l1(np.zeros((0, 3)), g["truth_pts"])
    with pytest.raises(ng.StructuralError):
        M.PointGrid(np.zeros((0, 3)))


def test_cameras_and_reference_render(env):
    ng, M, tor, fld, g = env
    cams = M.fibonacci_cameras(5, width=48, height=40)
    np.testing.assert_array_equal(np.stack([c.position for c in cams]), g["fib_pos"])
    np.testing.assert_array_equal(np.stack([c.up for c in cams]), g["fib_up"])
    h, n, ok = M.render_reference(cams[0], tor)
    assert _agree(h, g["ref_hit"]) >= HIT_AGREE
    both = ok & g["ref_ok"]
    assert both.sum() > 50
    np.testing.assert_allclose(n[both], g["ref_normal"][both], atol=1e-4)


def test_image_metrics_and_accuracy(env):
    ng, M, tor, fld, g = env
    iiou, nl2 = M.image_metrics(fld, tor, n_cameras=3, resolution=48)
    assert iiou == pytest.approx(float(g["iiou"]), abs=0.5)
    assert nl2 == pytest.approx(float(g["normal_l2"]), rel=0.05, abs=1e-4)
    acc = M.surface_accuracy(fld, tor, 300, 6, 4.0)
    assert acc == pytest.approx(float(g["accuracy"]), rel=0.1, abs=0.05)
    with pytest.raises(ng.ConfigError):
        M.image_metrics(fld, tor, n_cameras=0)


def test_bench_frame_and_csv(env, tmp_path):
    ng, M, tor, fld, g = env
    cam = ng.Camera((0.0, 2.0, 3.5), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 30.0, 32, 32)
    rows = M.bench_frame(fld, cam, [32, 64], lods=[2.5, 4], runs=5)
    assert [r.resolution for r in rows] == [32, 64, 32, 64]
    assert rows[1].pixels > rows[0].pixels and all(r.ms_trace > 0 for r in rows)
    M.write_bench_csv(tmp_path / "b.csv", rows)
    lines = (tmp_path / "b.csv").read_text().strip().splitlines()
    assert lines[0] == "resolution,pixels,ms_trace,ms_normals,evals,lod" and len(lines) == 5
    with pytest.raises(ng.ConfigError):
        M.bench_frame(fld, cam, [32], runs=4)
