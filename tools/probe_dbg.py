"""Debug: fused normal probes vs the separate normals pass on small frames."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2101_10994_b200 as ng
from paper_2101_10994_b200 import scenes
import importlib
R = importlib.import_module("paper_2101_10994_b200.render")
g = dict(np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/octree.npz")))
tor = scenes.Torus(0.5, 0.2)
svo = ng.build_octree(tor, 4, g["samples_b"])
fld = scenes.planted_field(svo, tor, seed=0, device_sdf=False)
for res in (32, 64):
    for lod in (2.5, 4.0):
        cam = ng.Camera((0.0, 2.0, 3.5), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 30.0, res, res)
        cfg = R.resolve_config(fld, ng.RenderConfig(lod=lod), lod)
        sess = R._session(fld, res, res)
        fr = sess.new_frame()
        sess.enqueue(cfg, fr, camera=cam)
        st = sess.read_stats()
        c = st.counters
        print(res, lod, "evals", c.decoder_evals, "nonfinite", c.nonfinite_inputs, "missing", c.evals_missing_level,
              "empty", c.empty_fallbacks, "visible", st.visible, "overflow", st.overflow,
              "normal_ok", int(fr["normal_ok"].sum()), "nan normals", int(fr["normal"].isnan().any(dim=1).sum()))
