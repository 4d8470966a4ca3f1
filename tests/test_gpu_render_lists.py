"""The render path's per-ray voxel lists at the BASELINE.json sizes, bit for
bit against the oracle's ray_trace_octree (traversal.py:207-247).

A frame's traversal (`k_traverse_tiles`, one warp per 32-ray tile, every
level in one launch) leaves its final (voxel, t_enter, t_exit) entries and
per-ray segments in the frame workspace; `RenderSession.final_list` reads
them back in the reference's order. The lists must equal the oracle's
final list in order, with t_enter / t_exit equal as fp64 bit patterns. The
near-tie slab decisions of the workload (within 2^-22 of flipping, the
fp32 scale) are counted and printed: an exact restatement agrees on every
one of them.

* configs[1]: torus-knot LOD5, 1280x720, every ray.
* configs[3]: torus-knot LOD6, 1920x1080, every 5th row.
* a band camera (the multi-GPU tiling): rank 1 of 3, its rays mapped back
  to global pixel indices.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bench_mod():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import bench
    return bench


def _frame_lists(ng, fld, cam, config, level):
    import sys
    R = sys.modules["paper_2101_10994_b200.render"]
    fb, rep = ng.render(cam, fld, config)
    sess = R._session(fld, cam.width, cam.height)
    fin, cells = sess.final_list(level, cells=True)
    st = sess.read_stats()
    n_levels = level + fld.svo.device.n_virtual
    assert len(fin) == int(st.pairs[n_levels])  # every claimed entry is in some ray's segment
    return fin, cells, rep


def _check_cells(svo, fin, cells, level):
    """The packed cell each tile-path entry carries is its voxel's cell."""
    from paper_2101_10994_b200.octree import morton_decode
    xyz = morton_decode(svo.levels[level].codes[fin.voxels]).astype(np.int64)
    packed = xyz[:, 0] | (xyz[:, 1] << 10) | (xyz[:, 2] << 20)
    assert np.array_equal(packed, cells)


def _report(name, r):
    print(f"\n{name}: {r['rays']} rays, {r['pairs']} final pairs, {r['decisions']} slab decisions, "
          f"{r['near_tie_decisions']} near-tie decisions (rel {r['tie_rel']:.2e}), "
          f"{r['mismatched_rays']} mismatched rays ({r['mismatched_near_tie']} with a near tie)")


def test_configs1_720p_lists_bit_exact(bench_mod):
    import paper_2101_10994_b200 as ng
    from oracle import nglod_oracle as O
    bench = bench_mod
    knot, svo, fld = bench.build_workload()
    c = bench.CAM
    cam = ng.Camera(c["position"], c["look_at"], c["up"], c["fov_y_deg"], bench.WIDTH, bench.HEIGHT)
    fin, cells, rep = _frame_lists(ng, fld, cam, ng.RenderConfig(), 5)
    _check_cells(svo, fin, cells, 5)
    tree = bench.oracle_tree(svo)
    o, d = O.camera_rays(c["position"], c["look_at"], c["up"], c["fov_y_deg"], bench.WIDTH, bench.HEIGHT)
    r = O.compare_final_lists(tree, o, d, fin.rays, fin.voxels, fin.t_enter, fin.t_exit, np.arange(len(o)), 5)
    _report("configs[1] 1280x720 LOD5", r)
    assert r["pairs"] == len(fin) and r["pairs"] > 3_000_000
    assert r["mismatched_rays"] == 0
    # the precondition under which the oracle's per-ray advance loop equals
    # the reference's batched one (render.py:202-238):
    # no voxel of the frame is entered beyond the far plane
    assert fin.t_enter.max() <= ng.RenderConfig().far_plane


def test_configs3_1080p_lod6_lists_bit_exact(bench_mod):
    import paper_2101_10994_b200 as ng
    from oracle import nglod_oracle as O
    from paper_2101_10994_b200 import scenes
    bench = bench_mod
    knot, samples = bench.knot_scene()
    svo6 = ng.build_octree(knot, 6, samples)
    fld6 = scenes.planted_field(svo6, knot, seed=0)
    c = bench.CAM
    cam = ng.Camera(c["position"], c["look_at"], c["up"], c["fov_y_deg"], 1920, 1080)
    fin, cells, rep = _frame_lists(ng, fld6, cam, ng.RenderConfig(), 6)
    _check_cells(svo6, fin, cells, 6)
    tree = bench.oracle_tree(svo6)
    o, d = O.camera_rays(c["position"], c["look_at"], c["up"], c["fov_y_deg"], 1920, 1080)
    rows = np.arange(2, 1080, 5)
    ids = (rows[:, None] * 1920 + np.arange(1920)[None, :]).ravel()
    r = O.compare_final_lists(tree, o, d, fin.rays, fin.voxels, fin.t_enter, fin.t_exit, ids, 6)
    _report("configs[3] 1920x1080 LOD6 (every 5th row)", r)
    assert r["pairs"] > 500_000
    assert r["mismatched_rays"] == 0
    assert fin.t_enter.max() <= ng.RenderConfig().far_plane  # the advance-loop precondition (see configs[1])


def test_band_camera_lists_bit_exact(bench_mod):
    """Rank 1 of 3 renders the 8-row bands b = 1, 4, 7, ...: its lists, with
    local ray ids mapped to global pixels, equal the oracle's for those rays."""
    import paper_2101_10994_b200 as ng
    from oracle import nglod_oracle as O
    from paper_2101_10994_b200.render import RenderSession, band_rows_of, resolve_config, resolve_lod
    bench = bench_mod
    knot, svo, fld = bench.build_workload()
    c = bench.CAM
    W, H = 640, 360
    cam = ng.Camera(c["position"], c["look_at"], c["up"], c["fov_y_deg"], W, H)
    rows = band_rows_of(H, 8, 3, 1)
    sess = RenderSession(fld, W, len(rows))
    config = ng.RenderConfig()
    cfg = resolve_config(fld, config, resolve_lod(cam, fld, config))
    n_levels = cfg.trace_level + svo.device.n_virtual
    import torch
    cs = cam.band_struct(8, 3, 1)
    while True:
        frame = sess.new_frame()
        from paper_2101_10994_b200 import _lib
        import ctypes
        _lib.call("ng_render_frame", svo.device.ref(), fld.device.ref(), ctypes.byref(cfg), ctypes.byref(cs),
                  ctypes.byref(sess.frame_struct(frame)), ctypes.byref(sess.ws), _lib.ptr(sess.stats),
                  _lib.stream_ptr())
        st = sess.read_stats()
        if not sess.grow(st, n_levels):
            break
    torch.cuda.synchronize()
    fin = sess.final_list(5)
    glob = (rows[:, None] * W + np.arange(W)[None, :]).ravel()
    o, d = O.camera_rays(c["position"], c["look_at"], c["up"], c["fov_y_deg"], W, H)
    r = O.compare_final_lists(bench.oracle_tree(svo), o, d, glob[fin.rays], fin.voxels, fin.t_enter, fin.t_exit,
                              glob, 5)
    _report("band camera rank 1/3 640x360", r)
    assert r["pairs"] > 10_000
    assert r["mismatched_rays"] == 0
