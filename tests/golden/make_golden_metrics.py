"""Generate the metrics golden fixtures from the REAL reference.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_metrics.py

Writes tests/golden/metrics.npz: the reference's metrics (octfield/metrics.py)
on the planted LOD4 torus of render.npz (octree 'b_' of octree.npz, planted
recipe of SURVEY.md Appendix A) -- oracle and field ray tracing, predicted
surface samples, signed extension, gIoU, Chamfer, nearest-neighbour
distances, Fibonacci cameras, the oracle reference render and the image
metrics. They pin paper_2101_10994_b200.metrics on the GPU box.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from octfield import field as F  # noqa: E402
from octfield import metrics as M  # noqa: E402
from octfield import octree as O  # noqa: E402
from octfield.geometry import AnalyticOracle, torus  # noqa: E402
from octfield.sampling import surface_points  # noqa: E402


def planted_torus(tor, samples):
    svo = O.build_octree(tor, 4, samples)
    fld = F.new_field(svo, seed=0)
    Z = fld.Z.copy()
    decs = [F.Decoder(d.W1.copy(), d.b1.copy(), d.W2.copy(), d.b2.copy()) for d in fld.decoders]
    for L in range(1, svo.max_level + 1):
        res = svo.resolution(L)
        ijk = O.morton_decode(svo.levels[L].codes)
        pos = (-1.0 + (ijk[:, None, :] + O.CORNER_OFFSETS[None]) * (2.0 / res)).reshape(-1, 3)
        Z[svo.levels[L].corners.ravel(), L - 1] = tor(pos).astype(np.float32)
        dd = decs[L - 1]
        dd.W1[0:2, :] = 0.0
        dd.b1[0:2] = 0.0
        dd.W1[0, 3 + L - 1] = 1.0
        dd.W1[1, 3 + L - 1] = -1.0
        dd.W2[:] = 0.0
        dd.W2[0, 0] = 1.0
        dd.W2[0, 1] = -1.0
        dd.b2[:] = 0.0
    return F.NeuralField(svo, Z, decs)


def main():
    tor = AnalyticOracle(torus(0.5, 0.2))
    samples = np.load(os.path.join(HERE, "octree.npz"))["samples_b"]
    fld = planted_torus(tor, samples)
    g = {}
    rays = M._random_rays(np.random.default_rng(1), 4096)
    g["rays_o"], g["rays_d"] = rays.origins, rays.directions
    g["oracle_hit"], g["oracle_t"] = M.trace_oracle_rays(tor, rays)
    g["field_hit"], g["field_t"] = M.trace_field_rays(fld, rays, 4.0)
    g["surf_pts"] = M.sample_predicted_surface(fld, 500, rng_seed=2, lod=4.0)
    pts = np.random.default_rng(3).uniform(-1.0, 1.0, size=(2000, 3))
    g["ext_pts"] = pts
    g["ext_l4"] = M.predict_signed_extension(fld, pts, 4)
    g["ext_l2"] = M.predict_signed_extension(fld, pts, 2)
    g["giou"] = np.float64(M.giou(fld, tor, 4096, rng_seed=4, level=4))
    truth = surface_points(tor, 500, 5)
    g["truth_pts"] = truth
    g["chamfer"] = np.float64(M.chamfer_l1(g["surf_pts"], truth))
    q = np.random.default_rng(6).uniform(-1.5, 1.5, size=(300, 3))
    g["nn_q"] = q
    g["nn_d"] = M.PointGrid(truth).nearest_dist(q)
    cams = M.fibonacci_cameras(5, width=48, height=40)
    g["fib_pos"] = np.stack([c.position for c in cams])
    g["fib_up"] = np.stack([c.up for c in cams])
    h, n, ok = M.render_reference(cams[0], tor)
    g["ref_hit"], g["ref_normal"], g["ref_ok"] = h, n, ok
    iiou, nl2 = M.image_metrics(fld, tor, n_cameras=3, resolution=48)
    g["iiou"], g["normal_l2"] = np.float64(iiou), np.float64(nl2)
    g["accuracy"] = np.float64(M.surface_accuracy(fld, tor, 300, 6, 4.0))
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **g)
    print("wrote metrics.npz:", {k: (v.shape if hasattr(v, "shape") else v) for k, v in g.items() if np.ndim(v) == 0})


if __name__ == "__main__":
    main()
