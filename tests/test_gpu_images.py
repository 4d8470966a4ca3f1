"""Device shading, threshold-LOD frames and the frame images against the
reference's golden fixtures (tests/golden/make_golden_images.py):
shade (render.py:303-314; test_render.py:328-337), render with
lod_thresholds (render.py:345-353; test_render.py:283-289), normal_image /
depth_image of our own frames (render.py:327-335; test_render.py:352-363)."""

import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DEPTH_TOL = 2e-3


@pytest.fixture(scope="module")
def ng():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2101_10994_b200 as pkg
    return pkg


def test_shade_golden_bit_exact(ng, golden):
    """ng_shade over 4,096 pixels (unit, non-unit, zero and axis normals; 70 % hits) equals the reference's u8."""
    g = golden("images")
    R = sys.modules["paper_2101_10994_b200.render"]
    got = R.shade(g["shade_hit"], g["shade_nrm"], ng.RenderConfig())
    assert got.shape == (64, 64, 3) and got.dtype == np.uint8
    np.testing.assert_array_equal(got, g["shade_default"])
    p = g["shade_cfg2_params"]
    cfg2 = ng.RenderConfig(light_dir=tuple(p[0:3]), albedo=tuple(p[3:6]), ambient=float(p[6]),
                           background=tuple(p[7:10]))
    np.testing.assert_array_equal(R.shade(g["shade_hit"], g["shade_nrm"], cfg2), g["shade_cfg2"])


def test_shade_midtones(ng):
    """test_render.py:328-337 restated."""
    R = sys.modules["paper_2101_10994_b200.render"]
    hit = np.array([[True, False]])
    nrm = np.zeros((1, 2, 3))
    nrm[0, 0] = [0.0, 1.0, 0.0]
    cfg = ng.RenderConfig()
    img = R.shade(hit, nrm, cfg)
    bg = (np.clip(np.asarray(cfg.background), 0, 1) * 255 + 0.5).astype(np.uint8)
    np.testing.assert_array_equal(img[0, 1], bg)
    assert img[0, 0].max() > bg.max()


@pytest.mark.parametrize("tag", ["th0", "th1"])
def test_threshold_lod_frames_golden(ng, golden, tag):
    """lod_thresholds select the reference's LOD (fractional 1.969 -> blend of levels 1, 2; and 4.0) and
    the frame matches the reference's at the north-star bars; the images of our frame match its images."""
    from paper_2101_10994_b200 import scenes
    from oracle import nglod_oracle as O
    R = sys.modules["paper_2101_10994_b200.render"]
    g = golden("images")
    go = golden("octree")
    svo = ng.build_octree(O.sdf_torus(0.5, 0.2), 4, go["samples_b"])
    fld = scenes.planted_field(svo, O.sdf_torus(0.5, 0.2), seed=0, device_sdf=False)
    cam = ng.Camera((0.0, 2.0, 3.5), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 30.0, 80, 60)
    fb, rep = ng.render(cam, fld, ng.RenderConfig(lod_thresholds=list(g[f"{tag}_th"])))
    assert rep.lod == float(g[f"{tag}_lod"])
    hit = g[f"{tag}_hit"]
    assert np.mean(fb.hit == hit) >= 0.999
    both = fb.hit & hit
    assert np.abs(fb.t[both] - g[f"{tag}_t"][both]).max(initial=0.0) <= DEPTH_TOL
    ev, vis = g[f"{tag}_report"]
    assert abs(rep.visible - vis) <= max(2, vis // 1000)
    assert abs(rep.evals - ev) <= max(10, ev // 100)
    same_px = np.all(fb.color == g[f"{tag}_color"], axis=-1)
    assert np.mean(same_px) >= 0.99, f"colour agreement {np.mean(same_px)}"
    # images of our frame: >= 99 % identical pixels; elsewhere within the normal bar (cos > 0.999: a few u8 steps)
    ni = R.normal_image(fb)
    assert ni.shape == (60, 80, 3) and ni.dtype == np.uint8
    assert np.all(ni[~fb.hit] == 0)
    diff = np.abs(ni.astype(int) - g[f"{tag}_normal_image"].astype(int))
    assert np.mean(np.all(diff == 0, axis=-1)) >= 0.99 and diff[both].max(initial=0) <= 8
    di = R.depth_image(fb, far=5.0)
    np.testing.assert_array_equal(di[..., 0], di[..., 2])
    ddiff = np.abs(di.astype(int) - g[f"{tag}_depth_image_5.0"].astype(int))
    assert ddiff[both].max(initial=0) <= 1 and np.all(di[~fb.hit] == 0)


def test_render_frames_equals_render(ng, golden):
    """render_frames (double-buffered readback) yields, frame by frame,
    exactly what render() returns; an overflowing first frame is grown and
    re-rendered before it is yielded."""
    from paper_2101_10994_b200 import scenes
    from oracle import nglod_oracle as O
    R = sys.modules["paper_2101_10994_b200.render"]
    go = golden("octree")
    svo = ng.build_octree(O.sdf_torus(0.5, 0.2), 4, go["samples_b"])
    fld = scenes.planted_field(svo, O.sdf_torus(0.5, 0.2), seed=0, device_sdf=False)
    cams = [ng.Camera((0.0, 2.0, 3.5), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 30.0, 96, 72),
            ng.Camera((2.5, 2.0, 2.0), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 35.0, 96, 72),
            ng.Camera((0.0, 2.0, 3.5), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 30.0, 96, 72)]
    cfg = ng.RenderConfig()
    want = [ng.render(c, fld, cfg) for c in cams]
    sess = R._session(fld, 96, 72)
    sess.pair_cap = sess.hit_cap = 64  # the first streamed frame overflows
    sess._alloc_ws()
    got = list(ng.render_frames(cams, fld, cfg))
    assert len(got) == len(cams)
    for (fb, rep), (fw, rw) in zip(got, want):
        for k in ("hit", "t", "normal", "normal_ok", "iterations", "evals", "color"):
            np.testing.assert_array_equal(getattr(fb, k), getattr(fw, k), err_msg=k)
        assert (rep.visible, rep.evals, rep.lod) == (rw.visible, rw.evals, rw.lod)
