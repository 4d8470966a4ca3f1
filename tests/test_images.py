"""Host-side frame helpers against the reference's golden fixtures
(tests/golden/make_golden_images.py): select_lod (render.py:140-152,
test_render.py:83-101), write_ppm (render.py:317-324, test_render.py:340-349),
normal_image / depth_image (render.py:327-335, test_render.py:352-363)
applied to the reference's own frame buffers. CPU only."""

import sys
import types

import numpy as np
import pytest

import paper_2101_10994_b200 as ng
import paper_2101_10994_b200.render  # noqa: F401
from paper_2101_10994_b200.errors import ConfigError, StructuralError

R = sys.modules["paper_2101_10994_b200.render"]  # the package re-exports render() over the module name


def _svo_stub(go, prefix):
    """select_lod reads only max_level and region."""
    region = types.SimpleNamespace(lo=go[prefix + "region_lo"], hi=go[prefix + "region_hi"])
    return types.SimpleNamespace(max_level=int(go[prefix + "max_level"]), region=region)


@pytest.mark.parametrize("tag,k", [("a", 0), ("a", 1), ("b", 0), ("b", 1)])
def test_select_lod_golden(golden, tag, k):
    g = golden("images")
    svo = _svo_stub(golden("octree"), tag + "_")
    th = list(g[f"lod_{tag}{k}_th"])
    got = np.array([ng.select_lod(ng.Camera(tuple(e), (0.0, 0.0, 0.0) if np.any(e[:2]) else (0.0, 0.0, e[2] - 1.0),
                                             (0.0, 1.0, 0.0), 30.0, 4, 4), svo, th) for e in g["lod_eyes"]])
    np.testing.assert_array_equal(got, g[f"lod_{tag}{k}"])  # bit-exact: same np.interp on the same distance


def test_select_lod_rejects_bad_thresholds(golden):
    svo = _svo_stub(golden("octree"), "a_")
    cam = ng.Camera((0.0, 0.0, 4.0), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 30.0, 4, 4)
    with pytest.raises(ConfigError):
        ng.select_lod(cam, svo, [1.0, 2.0])
    with pytest.raises(ConfigError):
        ng.select_lod(cam, svo, [1.0, 1.0, 2.0])


def test_write_ppm_golden(golden, tmp_path):
    g = golden("images")
    p = tmp_path / "x.ppm"
    ng.write_ppm(p, g["ppm_image"])
    assert p.read_bytes() == g["ppm_bytes"].tobytes()
    with pytest.raises(StructuralError):
        ng.write_ppm(p, g["ppm_image"].astype(np.float64))
    with pytest.raises(StructuralError):
        ng.write_ppm(p, g["ppm_image"][..., :2])


@pytest.mark.parametrize("tag", ["th0", "th1"])
def test_normal_and_depth_images_golden(golden, tag):
    """The image helpers on the reference's own frame buffer reproduce its images byte for byte."""
    g = golden("images")
    h, w = g[f"{tag}_hit"].shape
    fb = types.SimpleNamespace(width=w, height=h, hit=g[f"{tag}_hit"], t=g[f"{tag}_t"], normal=g[f"{tag}_normal"])
    np.testing.assert_array_equal(R.normal_image(fb), g[f"{tag}_normal_image"])
    for far in (5.0, 4.2):
        np.testing.assert_array_equal(R.depth_image(fb, far=far), g[f"{tag}_depth_image_{far}"])
