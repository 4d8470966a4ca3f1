"""Frame batches (ng_render_batch; render_batch, render_frames(batch=K),
TiledRenderer(batch=K)): several cameras in one traversal + one march, each
frame equal to render()'s for its camera in every per-pixel output."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELDS = ("hit", "t", "normal", "normal_ok", "iterations", "evals", "color")


@pytest.fixture(scope="module")
def ng():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2101_10994_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def torus(ng, golden):
    from paper_2101_10994_b200 import scenes
    from oracle import nglod_oracle as O
    go = golden("octree")
    svo = ng.build_octree(O.sdf_torus(0.5, 0.2), 4, go["samples_b"])
    return scenes.planted_field(svo, O.sdf_torus(0.5, 0.2), seed=0, device_sdf=False)


def _cams(ng, w=96, h=72):
    # distinct eye positions and fields of view: each frame its own camera
    return [ng.Camera((0.0, 2.0, 3.5), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 30.0, w, h),
            ng.Camera((2.5, 2.0, 2.0), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 35.0, w, h),
            ng.Camera((-1.0, -2.5, 2.5), (0.1, 0.0, 0.0), (0.0, 0.0, 1.0), 40.0, w, h),
            ng.Camera((0.3, 0.2, 0.4), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 60.0, w, h)]  # eye inside the octree


def _same(fb, fw):
    for k in FIELDS:
        np.testing.assert_array_equal(getattr(fb, k), getattr(fw, k), err_msg=k)


@pytest.mark.parametrize("config", ["default", "blend_shadows"])
def test_render_batch_equals_render(ng, torus, config):
    """Four cameras in one launch sequence: every frame equals render()'s bit for bit (camera rays, traversal
    lists, march, in-march normals and shading; with the LOD blend and shadow rays too); the batch report's
    totals are the frames' sums."""
    cfg = ng.RenderConfig() if config == "default" else ng.RenderConfig(lod=3.5, shadows=True)
    cams = _cams(ng)
    want = [ng.render(c, torus, cfg) for c in cams]
    fbs, rep = ng.render_batch(cams, torus, cfg)
    assert len(fbs) == len(cams)
    for fb, (fw, _) in zip(fbs, want):
        _same(fb, fw)
    assert rep.visible == sum(r.visible for _, r in want)
    assert rep.evals == sum(r.evals for _, r in want)
    if config != "default":
        assert rep.shadowed == sum(r.shadowed for _, r in want)
        assert rep.shadowed > 0


def test_render_batch_one_camera_and_limits(ng, torus):
    """A batch of one is render(); the launch maximum (NG_MAX_BATCH cameras) works; one more, mixed sizes and
    cameras whose automatic detail levels differ are ConfigErrors."""
    cams = _cams(ng)
    cfg = ng.RenderConfig()
    fbs, _ = ng.render_batch(cams[:1], torus, cfg)
    _same(fbs[0], ng.render(cams[0], torus, cfg)[0])
    from paper_2101_10994_b200 import _lib
    full = (cams * 8)[:_lib.MAX_BATCH]
    fbs, _ = ng.render_batch(full, torus, cfg)
    for fb, c in zip(fbs, full):
        _same(fb, ng.render(c, torus, cfg)[0])
    with pytest.raises(ng.ConfigError):
        ng.render_batch(cams * 8 + cams[:1], torus, cfg)
    with pytest.raises(ng.ConfigError):
        ng.render_batch([cams[0], ng.Camera((0.0, 2.0, 3.5), (0, 0, 0), (0, 1, 0), 30.0, 64, 48)], torus, cfg)
    th = ng.RenderConfig(lod_thresholds=(1.0, 2.0, 3.0, 6.0))
    near = ng.Camera((0.0, 0.5, 1.2), (0, 0, 0), (0, 1, 0), 30.0, 96, 72)
    far = ng.Camera((0.0, 2.0, 5.5), (0, 0, 0), (0, 1, 0), 30.0, 96, 72)
    with pytest.raises(ng.ConfigError):
        ng.render_batch([near, far], torus, th)


def test_render_frames_batched_equals_render(ng, torus):
    """render_frames(batch=3) over five cameras (a batch of three, then two; a detail-level change splits a
    batch) yields render()'s frames in order; an overflowing first batch is grown and re-rendered."""
    R = sys.modules["paper_2101_10994_b200.render"]
    cams = _cams(ng) + [_cams(ng)[1]]
    cfg = ng.RenderConfig()
    want = [ng.render(c, torus, cfg)[0] for c in cams]
    sess = R._session(torus, 96, 72, 3)
    sess.pair_cap = sess.hit_cap = 64  # the first batch overflows
    sess._alloc_ws()
    got = list(ng.render_frames(cams, torus, cfg, batch=3))
    assert len(got) == len(cams)
    for (fb, _), fw in zip(got, want):
        _same(fb, fw)
    th = ng.RenderConfig(lod_thresholds=(1.0, 2.0, 3.0, 6.0))
    near = ng.Camera((0.0, 0.5, 1.2), (0, 0, 0), (0, 1, 0), 30.0, 96, 72)
    far = ng.Camera((0.0, 2.0, 5.5), (0, 0, 0), (0, 1, 0), 30.0, 96, 72)
    seq = [near, near, far, far]
    got = list(ng.render_frames(seq, torus, th, batch=4))
    for (fb, rep), c in zip(got, seq):
        fw, rw = ng.render(c, torus, th)
        _same(fb, fw)
        assert rep.lod == rw.lod


def test_tiled_renderer_batch(ng, torus):
    """TiledRenderer(batch=3) on one rank: render_batch's images and per-pixel outputs are each frame's
    render() outputs, as (K, H, W, ...) device tensors."""
    from paper_2101_10994_b200.parallel import TiledRenderer
    cams = _cams(ng)[:3]
    cfg = ng.RenderConfig()
    t = TiledRenderer(torus, 96, 72, batch=3)
    imgs, visible, evals = t.render_batch(cams, cfg)
    assert tuple(imgs.shape) == (3, 72, 96, 3)
    want = [ng.render(c, torus, cfg) for c in cams]
    for f, (fw, _) in enumerate(want):
        np.testing.assert_array_equal(imgs[f].cpu().numpy(), fw.color)
    assert visible == sum(r.visible for _, r in want)
    out, _, _ = t.render_batch(cams, cfg, fields=("t", "hit"))
    for f, (fw, _) in enumerate(want):
        np.testing.assert_array_equal(out["t"][f].cpu().numpy(), fw.t)
        np.testing.assert_array_equal(out["hit"][f].cpu().numpy().astype(bool), fw.hit)
    img, _, _ = t.render(cams[1], cfg)  # one camera through a batch renderer
    np.testing.assert_array_equal(img.cpu().numpy(), want[1][0].color)


def test_batch_configs1_frame(ng):
    """configs[1] at full size in a batch with a second, orbiting camera: frame 0 is the benchmark frame
    (the reference's 112,420 visible pixels) and equals render(); frame 1 equals its own render()."""
    import bench
    import math
    knot, svo, fld = bench.build_workload()
    c0 = ng.Camera(bench.CAM["position"], bench.CAM["look_at"], bench.CAM["up"], bench.CAM["fov_y_deg"],
                   bench.WIDTH, bench.HEIGHT)
    a = math.radians(20.0)
    p = bench.CAM["position"]
    c1 = ng.Camera((p[0] * math.cos(a) + p[2] * math.sin(a), p[1], -p[0] * math.sin(a) + p[2] * math.cos(a)),
                   bench.CAM["look_at"], bench.CAM["up"], bench.CAM["fov_y_deg"], bench.WIDTH, bench.HEIGHT)
    cfg = ng.RenderConfig()
    fbs, rep = ng.render_batch([c0, c1], fld, cfg)
    f0, r0 = ng.render(c0, fld, cfg)
    f1, r1 = ng.render(c1, fld, cfg)
    assert int(fbs[0].hit.sum()) == 112420 == r0.visible
    _same(fbs[0], f0)
    _same(fbs[1], f1)
    assert rep.visible == r0.visible + r1.visible


@pytest.mark.parametrize("knobs", [{"NG_TILE_TRAVERSE": "0"}, {"NG_FUSED_PROBES": "0"},
                                   {"NG_TILE_SPLIT": "2", "NG_TILE_SPLIT_AHEAD": "1000000"},
                                   {"NG_TILE_SCAP": "3"}],
                         ids=["level_traversal", "normals_pass", "split_every_tile", "spill"])
def test_batch_under_knobs(ng, knobs):
    """The other code paths a batch can take (the level-by-level traversal with explicit per-frame camera
    rays and no shared eye, the separate normals pass, continuations on every tile, the shared-memory
    spill) give each frame render()'s outputs too (tests/batch_knob_probe.py in a subprocess: the knobs
    are read once per process)."""
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, os.path.join(here, "batch_knob_probe.py")], env={**os.environ, **knobs},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-3000:]
