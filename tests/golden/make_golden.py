"""Generate golden fixtures from the REAL reference package.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `octfield` from /root/reference/pkg/src, runs the hot-path
functions on small seeded inputs, and writes compressed .npz fixtures next
to this script. The fixtures pin the oracle (tests/test_oracle.py) and the
CUDA path (tests/test_gpu_*.py) on machines without the reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import octfield  # noqa: E402
from octfield import field as F  # noqa: E402
from octfield import octree as O  # noqa: E402
import octfield.render  # noqa: E402,F401
R = sys.modules["octfield.render"]
from octfield import traversal as T  # noqa: E402
from octfield.geometry import AnalyticOracle, sphere, torus  # noqa: E402
from octfield.sampling import build_epoch_set, surface_points  # noqa: E402


def svo_arrays(prefix, svo):
    out = {
        f"{prefix}r0": np.int64(svo.r0),
        f"{prefix}max_level": np.int64(svo.max_level),
        f"{prefix}corner_count": np.int64(svo.corner_count),
        f"{prefix}corner_offsets": svo.corner_offsets,
        f"{prefix}region_lo": svo.region.lo,
        f"{prefix}region_hi": svo.region.hi,
        f"{prefix}n_virtual": np.int64(len(svo.virtual_codes)),
    }
    for i, vc in enumerate(svo.virtual_codes):
        out[f"{prefix}vcodes{i}"] = vc
    for lv, L in enumerate(svo.levels):
        out[f"{prefix}codes{lv}"] = L.codes
        out[f"{prefix}parents{lv}"] = L.parents
        if L.corners is not None:
            out[f"{prefix}corners{lv}"] = L.corners
    return out


def test_rays(n, seed):
    """Acceptance crit-3 ray classes (test_acceptance.py:81-91)."""
    rng = np.random.default_rng(seed)
    origins = rng.uniform(-1.5, 1.5, size=(n, 3))
    dirs = rng.standard_normal((n, 3))
    dirs[:100, 0] = 0.0
    dirs[100:150, :2] = 0.0
    norms = np.linalg.norm(dirs, axis=1, keepdims=True)
    bad = norms[:, 0] < 1e-12
    dirs[bad] = (0.0, 0.0, 1.0)
    norms[bad] = 1.0
    return origins, dirs / norms


def f32pts(p):
    """fp32-representable float64 inputs."""
    return np.asarray(p, dtype=np.float32).astype(np.float64)


def main():
    sph = AnalyticOracle(sphere(0.5))
    tor = AnalyticOracle(torus(0.5, 0.2))

    # ---------------------------------------------------------------- morton
    rng = np.random.default_rng(0)
    ijk = rng.integers(0, 2**21, size=(4096, 3), dtype=np.int64)
    g = {"ijk": ijk, "codes": O.morton_encode(ijk)}
    np.savez_compressed(os.path.join(HERE, "morton.npz"), **g)

    # ---------------------------------------------------------------- octrees
    g = {}
    rng = np.random.default_rng(30)
    dirs = rng.standard_normal((4096, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    samples_a = f32pts(0.5 * dirs)
    svo_a = O.build_octree(sph, 3, samples_a)
    g["samples_a"] = samples_a
    g.update(svo_arrays("a_", svo_a))

    samples_b = f32pts(surface_points(tor, 4096, rng_seed=2))
    svo_b = O.build_octree(tor, 4, samples_b)
    g["samples_b"] = samples_b
    g.update(svo_arrays("b_", svo_b))

    samples_c = np.array([[0.9, 0.9, 0.9], [-0.9, -0.9, -0.9], [0.3, 0.3, 0.3]])
    svo_c = O.build_octree(None, 2, samples_c, corner_test=False)
    g["samples_c"] = samples_c
    g.update(svo_arrays("c_", svo_c))

    # corner-test-only lattice on the sphere at level 1 (test_octree.py:100-121)
    svo_d = O.build_octree(sph, 1, np.zeros((1, 3)), corner_test=True)
    g.update(svo_arrays("d_", svo_d))
    np.savez_compressed(os.path.join(HERE, "octree.npz"), **g)

    # ---------------------------------------------------------------- locate
    rng = np.random.default_rng(10)
    pts = f32pts(rng.uniform(-1.0, 1.0, size=(10_000, 3)))
    g = {"pts": pts}
    for lv in range(svo_a.max_level + 1):
        g[f"a_loc{lv}"] = O.locate(svo_a, pts, lv)
    # faces and the domain max (half-open binning, octree.py:134-139)
    edge_pts = np.array([[0.0, 0.0, 0.0], [1.0, 1.0, 1.0], [-1.0, -1.0, -1.0],
                         [0.5, -0.25, 0.125], [0.25, 0.25, 0.25]])
    g["edge_pts"] = edge_pts
    for lv in range(svo_a.max_level + 1):
        g[f"a_edge_loc{lv}"] = O.locate(svo_a, edge_pts, lv)
    np.savez_compressed(os.path.join(HERE, "locate.npz"), **g)

    # ---------------------------------------------------------------- slab
    rng = np.random.default_rng(21)
    n = 6_000
    o = rng.uniform(-3.0, 3.0, size=(n, 3))
    d = rng.standard_normal((n, 3))
    d[:1000, 0] = 0.0
    d[:500, 1] = 0.0
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    lo = rng.uniform(-1.0, 0.5, size=(n, 3))
    hi = lo + rng.uniform(0.05, 1.0, size=(n, 3))
    te, tx, hit = O.ray_aabb_batch(o, d, lo, hi)
    np.savez_compressed(os.path.join(HERE, "slab.npz"), o=o, d=d, lo=lo, hi=hi,
                        t_enter=te, t_exit=tx, hit=hit)

    # ---------------------------------------------------------------- traversal
    g = {}
    o, d = test_rays(1000, 11)
    g["o"], g["d"] = o, d
    for tag, svo in (("a", svo_a), ("b", svo_b)):
        lists = T.ray_trace_octree(T.RayBundle(o, d), svo, svo.max_level)
        g[f"{tag}_nlists"] = np.int64(len(lists))
        for i, lst in enumerate(lists):
            g[f"{tag}_L{i}_level"] = np.int64(lst.level)
            g[f"{tag}_L{i}_rays"] = lst.rays
            g[f"{tag}_L{i}_voxels"] = lst.voxels
        g[f"{tag}_t_enter"] = lists[-1].t_enter
        g[f"{tag}_t_exit"] = lists[-1].t_exit
        # a coarser target level
        lists2 = T.ray_trace_octree(T.RayBundle(o, d), svo, 2)
        g[f"{tag}_lvl2_rays"] = lists2[-1].rays
        g[f"{tag}_lvl2_voxels"] = lists2[-1].voxels
        g[f"{tag}_lvl2_t_enter"] = lists2[-1].t_enter
    rng = np.random.default_rng(31)
    scan_in = rng.integers(0, 2**40, size=5000, dtype=np.int64)
    g["scan_in"] = scan_in
    g["scan_out"] = T.exclusive_sum(scan_in)
    np.savez_compressed(os.path.join(HERE, "traversal.npz"), **g)

    # ---------------------------------------------------------------- field
    g = {}
    fld = F.new_field(svo_a, seed=0)
    g["Z_sum"] = np.float64(fld.Z.astype(np.float64).sum())
    g["Z_row7"] = fld.Z[7]
    for L, dec in enumerate(fld.decoders, start=1):
        g[f"W1_{L}"], g[f"b1_{L}"], g[f"W2_{L}"], g[f"b2_{L}"] = dec.W1, dec.b1, dec.W2, dec.b2
    ep = build_epoch_set(sph, 2000, rng_seed=5)
    pts = f32pts(ep.points)
    g["pts"] = pts
    for L in (1, 2, 3):
        c = F.EvalCounter()
        g[f"predict{L}"] = F.predict(svo_a, fld.Z, fld.decoders, pts, L, c)
        g[f"predict{L}_counts"] = np.array([c.decoder_evals, c.evals_missing_level, c.empty_fallbacks])
        out, _ = F.forward(svo_a, fld.Z, fld.decoders, pts, L)
        g[f"forward{L}"] = out
    for lt in (0.5, 1.75, 2.5):
        c = F.EvalCounter()
        g[f"blend{lt}"] = F.blend(svo_a, fld.Z, fld.decoders, pts, lt, c)
        g[f"blend{lt}_counts"] = np.array([c.decoder_evals, c.evals_missing_level, c.empty_fallbacks])
    z, mask = F.sum_features(svo_a, fld.Z, pts[:300], 3)
    g["sum3_z"], g["sum3_mask"] = z, mask
    psi, m2 = F.trilinear(svo_a, fld.Z, pts[:300], 2)
    g["tri2_psi"], g["tri2_mask"] = psi, m2
    g["empty"] = F.empty_space_value(svo_a, pts[:300])
    np.savez_compressed(os.path.join(HERE, "field.npz"), **g)

    # ---------------------------------------------------------------- render
    g = {}
    # cfg1-style: random-init sphere field (degenerate: first-eval hits)
    cam1 = R.Camera((0.0, 0.0, 4.0), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 30.0, 64, 64)
    fb, rep = R.render(cam1, fld, R.RenderConfig())
    for k in ("hit", "t", "iterations", "evals", "normal", "normal_ok", "color"):
        g[f"s_{k}"] = getattr(fb, k)
    g["s_report"] = np.array([rep.evals, rep.visible])
    o1 = cam1.rays()
    g["s_dirs"] = o1.directions

    # planted torus, LOD 4, off-axis camera
    fld_t = F.new_field(svo_b, seed=0)
    Z = fld_t.Z.copy()
    decs = [F.Decoder(dd.W1.copy(), dd.b1.copy(), dd.W2.copy(), dd.b2.copy()) for dd in fld_t.decoders]
    for L in range(1, svo_b.max_level + 1):
        res = svo_b.resolution(L)
        ijk = O.morton_decode(svo_b.levels[L].codes)
        pos = (-1.0 + (ijk[:, None, :] + O.CORNER_OFFSETS[None]) * (2.0 / res)).reshape(-1, 3)
        Z[svo_b.levels[L].corners.ravel(), L - 1] = tor(pos).astype(np.float32)
        dd = decs[L - 1]
        dd.W1[0:2, :] = 0.0
        dd.b1[0:2] = 0.0
        dd.W1[0, 3 + L - 1] = 1.0
        dd.W1[1, 3 + L - 1] = -1.0
        dd.W2[:] = 0.0
        dd.W2[0, 0] = 1.0
        dd.W2[0, 1] = -1.0
        dd.b2[:] = 0.0
    planted = F.NeuralField(svo_b, Z, decs)
    g["t_Z_sum"] = np.float64(Z.astype(np.float64).sum())
    cam2 = R.Camera((0.0, 2.0, 3.5), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 30.0, 96, 72)
    for tag, lod in (("t", None), ("f", 3.5)):
        fb, rep = R.render(cam2, planted, R.RenderConfig(lod=lod))
        for k in ("hit", "t", "iterations", "evals", "normal", "normal_ok", "color"):
            g[f"{tag}_{k}"] = getattr(fb, k)
        g[f"{tag}_report"] = np.array([rep.evals, rep.visible])
    np.savez_compressed(os.path.join(HERE, "render.npz"), **g)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
