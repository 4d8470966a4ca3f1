"""Parity at the BASELINE.json sizes (the bench workloads), checked against
the CPU oracle on bounded row / point samples.

* configs[1]: torus-knot LOD5 octree (device lattice), planted field,
  1280x720. The full frame is rendered; every 8th row is compared with the
  oracle. SURVEY.md section 6 measured this scene with the real reference:
  112,420 visible pixels and 1,425,674 decoder evaluations.
* configs[2]: batched query, 2^24 points. All points are evaluated, and 8,192
  random rows are compared with the oracle's forward (<= 1e-4).
* configs[3] / [4]: LOD6 at 1920x1080, integer LOD and LOD 4.5 with shadow
  rays. Every 18th / 36th row is compared with the oracle.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SDF_TOL = 1e-4
DEPTH_TOL = 2e-3


@pytest.fixture(scope="module")
def work():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import bench
    knot, svo, fld = bench.build_workload()
    return bench, knot, svo, fld


def _compare_rows(bench, ng, O, fld, tree, width, height, cam, config, params, stride, offset=0):
    fb, rep = ng.render(ng.Camera(cam["position"], cam["look_at"], cam["up"], cam["fov_y_deg"], width, height),
                        fld, config)
    rows = np.arange(offset, height, stride)
    idx = (rows[:, None] * width + np.arange(width)[None, :]).ravel()
    decs = [O.OracleDecoder(d.W1, d.b1, d.W2, d.b2) for d in fld.decoders]
    fr = O.render(tree, fld.Z, decs, dict(cam, width=width, height=height), params, ray_slice=idx,
                  workers=os.cpu_count() or 1)
    hit = fb.hit.reshape(-1)[idx]
    assert np.mean(hit == fr.hit) >= 0.999
    both = hit & fr.hit
    assert both.sum() > 1000
    assert np.max(np.abs(fb.t.reshape(-1)[idx][both] - fr.t[both])) <= DEPTH_TOL
    col = fb.color.reshape(-1, 3)[idx]
    assert np.mean(np.all(col == fr.color, axis=-1)) >= 0.99
    return fb, rep, fr


def test_configs1_720p_frame(work):
    bench, knot, svo, fld = work
    import paper_2101_10994_b200 as ng
    from oracle import nglod_oracle as O
    tree = bench.oracle_tree(svo)
    fb, rep, fr = _compare_rows(bench, ng, O, fld, tree, bench.WIDTH, bench.HEIGHT, bench.CAM, ng.RenderConfig(),
                                O.RenderParams(), stride=8)
    # known answer of the real reference on this scene
    assert rep.visible == 112420
    assert rep.evals == 1425674 or abs(rep.evals - 1425674) <= 20  # near-threshold fp32 iteration flips


def test_configs2_query_2e24(work):
    bench, knot, svo, fld = work
    import torch
    from oracle import nglod_oracle as O
    from paper_2101_10994_b200.field import forward_levels_device
    pts_h = bench.query_points(knot, bench.QUERY_POINTS)
    out = forward_levels_device(svo, fld.device, torch.from_numpy(pts_h).cuda(), [1, 2, 3, 4, 5]).cpu().numpy()
    assert out.shape == (bench.QUERY_POINTS, 5) and np.all(np.isfinite(out))
    rows = np.random.default_rng(0).choice(bench.QUERY_POINTS, 8192, replace=False)
    tree = bench.oracle_tree(svo)
    decs = [O.OracleDecoder(d.W1, d.b1, d.W2, d.b2) for d in fld.decoders]
    ref = O.forward_levels(tree, fld.Z, decs, pts_h[rows], [1, 2, 3, 4, 5])
    np.testing.assert_allclose(out[rows], ref, atol=SDF_TOL, rtol=0)
    # the public host-array call (chunked, pipelined through pinned staging)
    # returns the device call's values bit for bit
    host = fld.forward_levels(pts_h, [1, 2, 3, 4, 5])
    np.testing.assert_array_equal(host, out)
    # a resident output buffer (out=) is written in place with the same values
    buf = torch.full((bench.QUERY_POINTS, 5), np.nan, dtype=torch.float64, device="cuda")
    ret = forward_levels_device(svo, fld.device, torch.from_numpy(pts_h).cuda(), [1, 2, 3, 4, 5], out=buf)
    assert ret is buf
    np.testing.assert_array_equal(buf.cpu().numpy(), out)
    from paper_2101_10994_b200.errors import StructuralError
    with pytest.raises(StructuralError):
        forward_levels_device(svo, fld.device, torch.from_numpy(pts_h[:10]).cuda(), [1, 2], out=buf)


def test_host_query_chunks_and_errors(work):
    """NeuralField.forward_levels on host arrays: ragged chunk counts, a
    column subset, empty input, an out-of-domain point in a later chunk
    (StructuralError, octree.py:268-269) and a NaN point (the device call's
    outcome)."""
    bench, knot, svo, fld = work
    import torch
    from paper_2101_10994_b200.errors import OctfieldError, StructuralError
    from paper_2101_10994_b200.field import HOST_CHUNK, forward_levels_device
    rng = np.random.default_rng(5)
    for n in (1, 1000, HOST_CHUNK, 2 * HOST_CHUNK + 12345):
        pts = rng.uniform(-1.0, 1.0, size=(n, 3))
        want = forward_levels_device(svo, fld.device, torch.from_numpy(pts).cuda(), [2, 5]).cpu().numpy()
        np.testing.assert_array_equal(fld.forward_levels(pts, [5, 2]), want)
    assert fld.forward_levels(np.zeros((0, 3)), [1]).shape == (0, 1)
    bad = rng.uniform(-1.0, 1.0, size=(HOST_CHUNK + 7, 3))
    bad[HOST_CHUNK + 3, 1] = 1.0 + 1e-12
    with pytest.raises(StructuralError):
        fld.forward_levels(bad, [1, 2])
    bad[HOST_CHUNK + 3, 1] = np.nan  # passes the domain test (as in the reference); same outcome as the device call
    try:
        want = forward_levels_device(svo, fld.device, torch.from_numpy(bad).cuda(), [1, 2]).cpu().numpy()
    except OctfieldError:
        with pytest.raises(OctfieldError):
            fld.forward_levels(bad, [1, 2])
    else:
        np.testing.assert_array_equal(fld.forward_levels(bad, [1, 2]), want)


@pytest.fixture(scope="module")
def lod6(work):
    bench, knot, svo, fld = work
    import paper_2101_10994_b200 as ng
    from paper_2101_10994_b200 import scenes
    _, samples = bench.knot_scene()
    svo6 = ng.build_octree(knot, 6, samples)
    return svo6, scenes.planted_field(svo6, knot, seed=0)


def test_configs3_lod6_1080p(work, lod6):
    bench = work[0]
    import paper_2101_10994_b200 as ng
    from oracle import nglod_oracle as O
    svo6, fld6 = lod6
    _compare_rows(bench, ng, O, fld6, bench.oracle_tree(svo6), 1920, 1080, bench.CAM, ng.RenderConfig(),
                  O.RenderParams(), stride=18, offset=7)


def test_configs4_lod45_shadows_1080p(work, lod6):
    bench = work[0]
    import paper_2101_10994_b200 as ng
    from oracle import nglod_oracle as O
    svo6, fld6 = lod6
    fb, rep, fr = _compare_rows(bench, ng, O, fld6, bench.oracle_tree(svo6), 1920, 1080, bench.CAM,
                                ng.RenderConfig(lod=4.5, shadows=True), O.RenderParams(lod=4.5, shadows=True),
                                stride=36, offset=3)
    assert fr.shadowed.sum() > 0


def test_configs0_sphere_lod3_128():
    """configs[0]: LOD1-3 octree of the analytic sphere, random-init field
    (feature dim 32, hidden 128), 128x128 frame, against the oracle's render
    of the same octree and field (the reference measured
    4,244 hits, all on the first evaluation, and 5,313 evaluations)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import bench
    import paper_2101_10994_b200 as ng
    from paper_2101_10994_b200 import scenes
    from oracle import nglod_oracle as O
    sphere = scenes.Sphere(0.5)
    svo = ng.build_octree(sphere, 3, ng.surface_points(sphere, 2 ** 17, 0))
    fld = ng.new_field(svo, seed=0)
    cam = dict(position=(0.0, 0.0, 4.0), look_at=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0), fov_y_deg=30.0)
    fb, rep = ng.render(ng.Camera(cam["position"], cam["look_at"], cam["up"], 30.0, 128, 128), fld,
                        ng.RenderConfig())
    decs = [O.OracleDecoder(d.W1, d.b1, d.W2, d.b2) for d in fld.decoders]
    fr = O.render(bench.oracle_tree(svo), fld.Z, decs, dict(cam, width=128, height=128), O.RenderParams(),
                  workers=8)
    print(f"\nconfigs[0]: {rep.visible} visible (oracle {fr.visible}), {rep.evals} evals (oracle {fr.total_evals}), "
          f"{int((fb.hit != fr.hit).sum())} hit pixels differ")
    assert fr.visible > 4000
    assert np.mean(fb.hit == fr.hit) >= 0.999
    both = fb.hit & fr.hit
    assert np.abs(fb.t[both] - fr.t[both]).max() <= DEPTH_TOL
    assert np.mean(np.all(fb.color == fr.color, axis=-1)) >= 0.999
    assert abs(rep.evals - fr.total_evals) <= max(10, fr.total_evals // 1000)
