"""The render path's warp-per-tile traversal (traverse.cu k_traverse_tiles)
against the level-by-level kernels and the golden frame, including its
shared-memory spill path and the overflow -> grow -> rerun loop; and the
normals evaluated inside the march against the separate normals pass. The knobs
are read once per process, so each configuration renders in a subprocess
(tests/tile_probe.py)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _probe(tmp_path, name, env, *args):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    out = str(tmp_path / f"{name}.npz")
    subprocess.run([sys.executable, os.path.join(HERE, "tile_probe.py"), out, *args], check=True,
                   env={**os.environ, **env}, timeout=600)
    return dict(np.load(out))


@pytest.fixture(scope="module")
def frames(tmp_path_factory):
    tmp = tmp_path_factory.mktemp("tiles")
    return {
        "tiles": _probe(tmp, "tiles", {}),
        "levels": _probe(tmp, "levels", {"NG_TILE_TRAVERSE": "0"}),
        "spill": _probe(tmp, "spill", {"NG_TILE_SCAP": "3"}),
        "overflow": _probe(tmp, "overflow", {"NG_TILE_SCAP": "0", "NG_TILE_ARENA_MIN": "0"}, "tiny_pairs"),
        "normals_pass": _probe(tmp, "normals_pass", {"NG_FUSED_PROBES": "0"}),
        # split every list longer than 2 entries from the first tile on
        # (continuations, the entry pool and the ticket queue on every tile)
        "split": _probe(tmp, "split", {"NG_TILE_SPLIT": "2", "NG_TILE_SPLIT_AHEAD": "1000000"}),
        "split_spill": _probe(tmp, "split_spill", {"NG_TILE_SPLIT": "2", "NG_TILE_SPLIT_AHEAD": "1000000",
                                                   "NG_TILE_SCAP": "3"}),
    }


def _same(a, b):
    for k in ("hit", "t", "color", "iterations", "evals", "visible", "n_evals", "normal", "normal_ok"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


def test_tiles_equal_level_by_level(frames):
    """Per-ray segments from the tile kernel drive the identical march."""
    _same(frames["tiles"], frames["levels"])


def test_tiles_match_golden_frame(frames, golden):
    g = golden("render")
    f = frames["tiles"]
    assert np.mean(f["hit"] == g["t_hit"]) >= 0.999
    ev, vis = g["t_report"]
    assert abs(int(f["visible"]) - vis) <= max(2, vis // 1000)


def test_spill_path_identical(frames):
    """Lists held almost entirely in the global arena give the same frame."""
    _same(frames["spill"], frames["tiles"])


def test_overflow_grows_and_reruns(frames):
    f = frames["overflow"]
    assert int(f["grows"]) >= 1
    _same(f, frames["tiles"])


def _same_lists(a, b):
    for k in ("l_rays", "l_voxels", "l_t_enter", "l_t_exit"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


def test_split_tiles_identical(frames):
    """Tiles split into continuations at ray boundaries (traverse.cu) give
    the same per-ray lists (order included) and the same frame, with the
    lists in shared memory or in the spill arena."""
    assert len(frames["tiles"]["l_rays"]) > 1000
    for k in ("split", "split_spill"):
        assert int(frames[k]["splits"]) > 10, f"{k}: no tile was split"
        _same_lists(frames[k], frames["tiles"])
        _same(frames[k], frames["tiles"])


def test_tile_lists_equal_level_by_level(frames):
    _same_lists(frames["tiles"], frames["levels"])


def test_probes_in_march_equal_normals_pass(frames):
    """Normals evaluated as probe items inside the march (default) equal the
    separate k_normals pass bit for bit (same evaluations, same counters)."""
    _same(frames["tiles"], frames["normals_pass"])


def _degenerate_rays():
    """Rays the tile traversal's fast test excludes (a zero direction
    component) or whose slab values tie: axis-aligned and diagonal
    directions from origins on the LOD4 lattice planes and edges."""
    rng = np.random.default_rng(11)
    h = 2.0 / 64  # LOD4 cell edge (res 64)
    o, d = [], []
    axes = [np.array(v, float) for v in [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]]
    diag = [np.array(v, float) / np.linalg.norm(v) for v in [(1, 1, 0), (1, -1, 0), (0, 1, -1), (1, 1, 1), (-1, 1, -1)]]
    for _ in range(1500):
        k = rng.integers(-40, 41, size=3)
        p = k * h  # lattice points and planes
        jitter = rng.uniform(-0.6, 0.6, size=3)
        mask = rng.integers(0, 2, size=3).astype(bool)
        p = np.where(mask, p, jitter)  # some coordinates on planes, others free
        dirs = axes + diag
        dv = dirs[rng.integers(0, len(dirs))]
        start = p - 1.7 * dv  # start outside the shape, travel through p
        o.append(start)
        d.append(dv)
    return np.array(o), np.array(d)


def test_degenerate_rays_match_oracle(golden):
    """Explicit rays through the render path (tile traversal with per-ray
    origins, both the ordered and the literal slab paths, then the march)
    against the oracle's traversal + march."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2101_10994_b200 as ng
    from paper_2101_10994_b200 import scenes
    from paper_2101_10994_b200.render import trace_rays
    from oracle import nglod_oracle as O
    from conftest import oracle_tree_from_golden
    go = golden("octree")
    svo = ng.build_octree(O.sdf_torus(0.5, 0.2), 4, go["samples_b"])
    tree = oracle_tree_from_golden(go, "b_")
    fld = scenes.planted_field(svo, O.sdf_torus(0.5, 0.2), seed=0, device_sdf=False)
    decs = [O.OracleDecoder(dd.W1, dd.b1, dd.W2, dd.b2) for dd in fld.decoders]
    o, d = _degenerate_rays()
    assert (d == 0).any(axis=1).sum() > 500  # many rays take the literal path
    hit, t = trace_rays(fld, ng.RayBundle(o, d), 4.0)
    ofin = O.traverse(tree, o, d, 4)[-1]
    ohit, ot, _, _ = O.march(tree, fld.Z, decs, o, d, ofin, 4.0, O.RenderParams())
    assert hit.sum() > 300
    assert np.mean(hit == ohit) >= 0.999
    both = hit & ohit
    assert np.abs(t[both] - ot[both]).max(initial=0.0) <= 2e-3
