"""Golden fixtures for the frame-level helpers around the hot path, from the
REAL reference package: select_lod (render.py:140-152), threshold-LOD
frames (render.py:345-353), shade (render.py:303-314), write_ppm
(render.py:317-324), normal_image / depth_image (render.py:327-335).

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_images.py

The octrees are rebuilt by the reference from the samples stored in
octree.npz (make_golden.py), so both fixture files describe the same trees.
"""

from __future__ import annotations

import io
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from octfield import field as F  # noqa: E402
from octfield import octree as O  # noqa: E402
import octfield.render  # noqa: E402,F401
R = sys.modules["octfield.render"]
from octfield.geometry import AnalyticOracle, sphere, torus  # noqa: E402


def planted(svo, oracle, seed=0):
    """SURVEY.md Appendix A planted field, as make_golden.py builds it."""
    fld = F.new_field(svo, seed=seed)
    Z = fld.Z.copy()
    decs = [F.Decoder(d.W1.copy(), d.b1.copy(), d.W2.copy(), d.b2.copy()) for d in fld.decoders]
    for L in range(1, svo.max_level + 1):
        res = svo.resolution(L)
        ijk = O.morton_decode(svo.levels[L].codes)
        pos = (-1.0 + (ijk[:, None, :] + O.CORNER_OFFSETS[None]) * (2.0 / res)).reshape(-1, 3)
        Z[svo.levels[L].corners.ravel(), L - 1] = oracle(pos).astype(np.float32)
        d = decs[L - 1]
        d.W1[0:2, :] = 0.0
        d.b1[0:2] = 0.0
        d.W1[0, 3 + L - 1] = 1.0
        d.W1[1, 3 + L - 1] = -1.0
        d.W2[:] = 0.0
        d.W2[0, 0] = 1.0
        d.W2[0, 1] = -1.0
        d.b2[:] = 0.0
    return F.NeuralField(svo, Z, decs)


def main():
    sph = AnalyticOracle(sphere(0.5))
    tor = AnalyticOracle(torus(0.5, 0.2))
    oct_npz = np.load(os.path.join(HERE, "octree.npz"))
    svo_a = O.build_octree(sph, 3, oct_npz["samples_a"])
    svo_b = O.build_octree(tor, 4, oct_npz["samples_b"])
    g = {}

    # ------------------------------------------------------------ select_lod
    # eye positions along three axes and off-axis, at distances that land
    # below, on, between and past the thresholds (test_render.py:83-101)
    rng = np.random.default_rng(40)
    eyes = np.concatenate([
        np.array([[0.0, 0.0, z] for z in np.linspace(0.2, 9.0, 45)]),
        rng.normal(size=(40, 3)) * 3.0,
    ])
    g["lod_eyes"] = eyes
    for tag, svo, ths in (("a", svo_a, ([1.0, 2.0, 3.0], [0.5, 2.25, 7.0])),
                          ("b", svo_b, ([1.0, 2.0, 3.0, 4.0], [2.0, 3.0, 4.0, 5.0]))):
        for k, th in enumerate(ths):
            g[f"lod_{tag}{k}_th"] = np.asarray(th)
            g[f"lod_{tag}{k}"] = np.array([R.select_lod(R.Camera(tuple(e), (0.0, 0.0, 0.0) if np.any(e[:2]) else
                                                                  (0.0, 0.0, e[2] - 1.0), (0.0, 1.0, 0.0), 30.0, 4, 4),
                                                         svo, th) for e in eyes])

    # ------------------------------------------------------ threshold frames
    fld_t = planted(svo_b, tor)
    cam = R.Camera((0.0, 2.0, 3.5), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 30.0, 80, 60)
    for tag, th in (("th0", [2.0, 3.0, 4.0, 5.0]), ("th1", [4.5, 5.0, 6.0, 7.0])):
        fb, rep = R.render(cam, fld_t, R.RenderConfig(lod_thresholds=th))
        g[f"{tag}_th"] = np.asarray(th)
        g[f"{tag}_lod"] = np.float64(rep.lod)
        for k in ("hit", "t", "iterations", "evals", "normal", "normal_ok", "color"):
            g[f"{tag}_{k}"] = getattr(fb, k)
        g[f"{tag}_report"] = np.array([rep.evals, rep.visible])
        g[f"{tag}_normal_image"] = R.normal_image(fb)
        for far in (5.0, 4.2):
            g[f"{tag}_depth_image_{far}"] = R.depth_image(fb, far=far)

    # ------------------------------------------------------------------ shade
    # unit normals over the sphere (every Lambert value from 0 to 1), the
    # axis-aligned cases of test_render.py:328-337, non-unit and zero rows
    n = 4096
    nrm = rng.normal(size=(n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    nrm[:6] = np.array([[1, 0, 0], [0, 1, 0], [0, 0, 1], [-1, 0, 0], [0, -1, 0], [0, 0, -1]], dtype=np.float64)
    nrm[6] = 0.0
    nrm[7:64] *= rng.uniform(0.0, 3.0, size=(57, 1))
    hit = rng.uniform(size=n) < 0.7
    hit[:8] = True
    g["shade_hit"] = hit.reshape(64, 64)
    g["shade_nrm"] = nrm.reshape(64, 64, 3)
    g["shade_default"] = R.shade(hit.reshape(64, 64), nrm.reshape(64, 64, 3), R.RenderConfig())
    cfg2 = R.RenderConfig(light_dir=(0.3, -0.2, 0.9), albedo=(0.9, 0.1, 0.5), ambient=0.3,
                          background=(0.0, 0.5, 1.2))
    g["shade_cfg2"] = R.shade(hit.reshape(64, 64), nrm.reshape(64, 64, 3), cfg2)
    g["shade_cfg2_params"] = np.array([*cfg2.light_dir, *cfg2.albedo, cfg2.ambient, *cfg2.background])

    # -------------------------------------------------------------- write_ppm
    img = rng.integers(0, 256, size=(7, 5, 3), dtype=np.uint8)
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "x.ppm")
        R.write_ppm(p, img)
        with open(p, "rb") as fh:
            g["ppm_bytes"] = np.frombuffer(fh.read(), dtype=np.uint8)
    g["ppm_image"] = img
    np.savez_compressed(os.path.join(HERE, "images.npz"), **g)
    print("images.npz written to", HERE)


if __name__ == "__main__":
    main()
