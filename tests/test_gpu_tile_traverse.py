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


def test_probes_in_march_equal_normals_pass(frames):
    """Normals evaluated as probe items inside the march (default) equal the
    separate k_normals pass bit for bit (same evaluations, same counters)."""
    _same(frames["tiles"], frames["normals_pass"])
