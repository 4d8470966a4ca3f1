"""Subprocess helper for tests/test_gpu_batch.py: with whatever NG_* knobs
the environment sets (read once per process), a batch of four distinct
cameras must equal render() per camera in every per-pixel output; exits 0
and prints "ok" when it does."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2101_10994_b200 as ng  # noqa: E402
from paper_2101_10994_b200 import scenes  # noqa: E402
from oracle import nglod_oracle as O  # noqa: E402

go = dict(np.load(os.path.join(ROOT, "tests", "golden", "octree.npz")))
svo = ng.build_octree(O.sdf_torus(0.5, 0.2), 4, go["samples_b"])
fld = scenes.planted_field(svo, O.sdf_torus(0.5, 0.2), seed=0, device_sdf=False)
cams = [ng.Camera((0.0, 2.0, 3.5), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 30.0, 96, 72),
        ng.Camera((2.5, 2.0, 2.0), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 35.0, 96, 72),
        ng.Camera((-1.0, -2.5, 2.5), (0.1, 0.0, 0.0), (0.0, 0.0, 1.0), 40.0, 96, 72),
        ng.Camera((0.3, 0.2, 0.4), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 60.0, 96, 72)]
for cfg in (ng.RenderConfig(), ng.RenderConfig(lod=3.5, shadows=True)):
    fbs, rep = ng.render_batch(cams, fld, cfg)
    vis = 0
    for fb, c in zip(fbs, cams):
        fw, rw = ng.render(c, fld, cfg)
        vis += rw.visible
        for k in ("hit", "t", "normal", "normal_ok", "iterations", "evals", "color"):
            assert np.array_equal(getattr(fb, k), getattr(fw, k), equal_nan=True), k
    assert rep.visible == vis > 0
print("ok")
