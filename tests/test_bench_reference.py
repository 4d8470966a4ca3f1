"""The reference arm's inputs and plumbing (bench.py --impl reference), on CPU.

The arm runs the unmodified reference package from baseline/_ref on inputs
the reference produced (bench_data/knot_l5_ref.npz, tools/make_ref_inputs.py).
These tests check that the rebuilt workload is configs[1] (voxel counts,
planted values against the knot SDF), that the row-sample composition of
the reference's render() yields the reference's traversal, and that both
arms describe the same config.
"""

import os

import numpy as np
import pytest

import bench


@pytest.fixture(scope="module")
def ref():
    r = bench.load_reference()
    if r is None:
        pytest.skip("reference not installed in baseline/_ref")
    return r


def test_ref_workload_is_configs1(ref):
    from paper_2101_10994_b200 import scenes
    svo, fld = bench.ref_workload(ref)
    assert [svo.voxel_count(lv) for lv in range(6)] == bench.VOXELS
    assert svo.corner_count == 117197
    knot = scenes.torus_knot(segments=1024, tube=0.08)
    rng = np.random.default_rng(0)
    for L in (1, 3, 5):
        lv = svo.levels[L]
        pick = rng.choice(len(lv.codes), 64, replace=False)
        res = svo.resolution(L)
        ijk = ref.octree.morton_decode(lv.codes[pick])
        pos = (-1.0 + (ijk[:, None, :] + ref.octree.CORNER_OFFSETS[None]) * (2.0 / res)).reshape(-1, 3)
        want = knot(pos).astype(np.float32)
        got = fld.Z[lv.corners[pick].ravel(), L - 1]
        assert np.array_equal(got, want)
        d = fld.decoders[L - 1]
        assert d.W1[0, 3 + L - 1] == 1.0 and d.W2[0, 0] == 1.0 and d.W2[0, 2:].max() == 0.0


def test_ref_row_sample_traversal_matches_oracle(ref):
    from oracle import nglod_oracle as O
    svo, fld = bench.ref_workload(ref)
    rows = np.array([250, 400])
    secs, n, fin, rep, idx = bench.ref_row_sample(ref, fld, rows, workers=2)
    assert n == 2 * bench.WIDTH and rep.visible > 0
    o, d = O.camera_rays(bench.CAM["position"], bench.CAM["look_at"], bench.CAM["up"], bench.CAM["fov_y_deg"],
                         bench.WIDTH, bench.HEIGHT)
    of = O.traverse(bench.oracle_tree(svo), o[idx], d[idx], 5)[-1]
    assert np.array_equal(of.rays, fin.rays) and np.array_equal(of.voxels, fin.voxels)
    assert np.array_equal(of.t_enter, fin.t_enter) and np.array_equal(of.t_exit, fin.t_exit)

    class Ours:  # the GPU side's list, with global ray ids
        rays = idx[of.rays]
        voxels = of.voxels
        t_enter = of.t_enter
        t_exit = of.t_exit
    assert bench.compare_lists(Ours, fin, idx, bench.WIDTH * bench.HEIGHT)["mismatched_rays"] == 0
    Ours.t_exit = np.nextafter(of.t_exit, 10.0)  # one ulp off everywhere
    assert bench.compare_lists(Ours, fin, idx, bench.WIDTH * bench.HEIGHT)["mismatched_rays"] > 0


def test_reference_arm_never_imports_the_package():
    """The reference arm's code path names only the reference and numpy."""
    import inspect
    src = "".join(inspect.getsource(f) for f in (bench.run_reference, bench.ref_workload, bench.ref_camera,
                                                  bench.load_reference, bench.Reference))
    assert "paper_2101_10994_b200" not in src and "oracle" not in src


def test_both_arms_share_the_config():
    assert bench.line_config(1) == bench.line_config(1)
    assert bench.line_config(2)["parallelism"].startswith("tiles2")
    assert os.path.exists(bench.REF_INPUTS)
