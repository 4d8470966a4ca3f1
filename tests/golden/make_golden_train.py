"""Generate the training-path golden fixtures from the REAL reference.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_train.py

Writes tests/golden/train.npz: the reference's epoch sample sets
(sampling.py), loss / gradients of loss_batch (trainer.py:106-144 through
field.backward, field.py:360-394), the hand-computed loss case
(test_trainer.py:54-79), Adam steps (trainer.py:87-103) and short training
runs for the joint, progressive and frozen-decoder schedules
(trainer.py:165-251). The fixtures pin oracle/train_oracle.py and the CUDA
training step on machines without the reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, HERE)

from make_golden import svo_arrays  # noqa: E402
from octfield import field as F  # noqa: E402
from octfield import trainer as T  # noqa: E402
from octfield.geometry import AnalyticOracle, sphere, torus  # noqa: E402
from octfield.octree import build_octree  # noqa: E402
from octfield.sampling import SampleSet, build_epoch_set, surface_points  # noqa: E402


def dec_arrays(prefix, decoders):
    out = {}
    for i, d in enumerate(decoders):
        out[f"{prefix}W1_{i}"] = d.W1
        out[f"{prefix}b1_{i}"] = d.b1
        out[f"{prefix}W2_{i}"] = d.W2
        out[f"{prefix}b2_{i}"] = d.b2
    return out


def grad_arrays(prefix, grads):
    out = {f"{prefix}dZ": grads.dZ}
    for i, g in enumerate(grads.decoders):
        out[f"{prefix}has{i}"] = np.int64(g is not None)
        if g is not None:
            out[f"{prefix}gW1_{i}"] = g.W1
            out[f"{prefix}gb1_{i}"] = g.b1
            out[f"{prefix}gW2_{i}"] = g.W2
            out[f"{prefix}gb2_{i}"] = g.b2
    return out


def main():
    g = {}
    sph = AnalyticOracle(sphere(0.5))

    # ---- tiny setup of test_trainer.py:24-29 (sphere, L=2, m=4, h=8)
    surf = surface_points(sph, 1024, rng_seed=0)
    svo = build_octree(sph, 2, surf)
    fld = F.new_field(svo, m=4, h=8, seed=0)
    g.update(svo_arrays("s_", svo))
    g["s_surf"] = surf
    g["s_Z"] = fld.Z
    g.update(dec_arrays("s_", fld.decoders))

    # ---- epoch sample set (sampling.py:177-196)
    ss = build_epoch_set(sph, 600, 10)
    g["ep_points"], g["ep_dist"], g["ep_tags"] = ss.points, ss.distances, ss.scheme_tags

    # ---- loss_batch + backward on the tiny field (active [1, 2]), fp64 work copy
    work = F.NeuralField(svo, fld.Z.astype(np.float64), [d.astype(np.float64) for d in fld.decoders])
    pts = surface_points(sph, 160, rng_seed=7)
    samples = SampleSet(pts, sph(pts), np.zeros(len(pts), np.int8))
    loss, grads, sums = T.loss_batch(work, samples, [1, 2])
    g["lb_pts"], g["lb_dist"] = pts, sph(pts)
    g["lb_loss"], g["lb_sums"] = np.float64(loss), sums
    g.update(grad_arrays("lb_", grads))
    loss2, grads2, sums2 = T.loss_batch(work, samples, [2])
    g["lb2_loss"], g["lb2_sums"] = np.float64(loss2), sums2
    g.update(grad_arrays("lb2_", grads2))

    # ---- the real widths: torus L3, m=32, h=128, epoch-mix points
    tor = AnalyticOracle(torus(0.5, 0.2))
    surf_t = surface_points(tor, 4096, rng_seed=1)
    svo_t = build_octree(tor, 3, surf_t)
    fld_t = F.new_field(svo_t, seed=3)
    g.update(svo_arrays("t_", svo_t))
    g["t_surf"] = surf_t
    g["t_Z"] = fld_t.Z
    g.update(dec_arrays("t_", fld_t.decoders))
    ep = build_epoch_set(tor, 512, 4)
    work_t = F.NeuralField(svo_t, fld_t.Z.astype(np.float64), [d.astype(np.float64) for d in fld_t.decoders])
    loss_t, grads_t, sums_t = T.loss_batch(work_t, ep, [1, 2, 3])
    g["tl_pts"], g["tl_dist"] = ep.points, ep.distances
    g["tl_loss"], g["tl_sums"] = np.float64(loss_t), sums_t
    g.update(grad_arrays("tl_", grads_t))

    # ---- Adam on the first gradient (trainer.py:87-103), two steps
    params = {"Z": work.Z.copy()}
    for i, d in enumerate(work.decoders):
        params[f"decoder{i + 1}.W1"] = d.W1.copy()
    st = T.AdamState.for_params(params)
    gd = {"Z": grads.dZ, "decoder2.W1": grads.decoders[1].W1}
    T.adam_step(params, gd, st, lr=0.01)
    T.adam_step(params, gd, st, lr=0.01)
    g["adam_Z"] = params["Z"]
    g["adam_W1_0"] = params["decoder1.W1"]
    g["adam_W1_1"] = params["decoder2.W1"]

    # ---- short training runs (test_trainer.py:193-268)
    runs = {
        "joint": T.TrainConfig(epochs=2, points_per_epoch=600, rng_seed=10),
        "prog": T.TrainConfig(epochs=3, points_per_epoch=500, schedule="progressive", progressive_interval=2,
                              rng_seed=14),
        "frozen": T.TrainConfig(epochs=2, points_per_epoch=700, schedule="frozen_decoder", rng_seed=16,
                                batch_size=200),
    }
    for tag, cfg in runs.items():
        out, hist = T.train(sph, fld, cfg)
        g[f"run_{tag}_Z"] = out.Z
        g.update(dec_arrays(f"run_{tag}_", out.decoders))
        g[f"run_{tag}_hist"] = np.stack([h.level_losses for h in hist])

    # ---- model file bytes (modelio.py:47-69) and a max_lod=1 load (modelio.py:140-151)
    import tempfile
    from octfield import modelio as M
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "tiny.nsdf")
        M.save_model(path, fld)
        with open(path, "rb") as fh:
            g["model_bytes"] = np.frombuffer(fh.read(), dtype=np.uint8).copy()
        cut = M.load_model(path, max_lod=1)
        g["cut_corner_count"] = np.int64(cut.svo.corner_count)
        g["cut_region_lo"], g["cut_region_hi"] = cut.svo.region.lo, cut.svo.region.hi
        g["cut_Z"] = cut.Z
        g["serialized_bytes"] = np.int64(M.serialized_bytes(fld))

    np.savez_compressed(os.path.join(HERE, "train.npz"), **g)
    print("wrote train.npz:", len(g), "arrays")


if __name__ == "__main__":
    main()
