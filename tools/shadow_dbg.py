"""Debug: shadow-ray determinism and agreement with the oracle composition."""
import sys, os, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2101_10994_b200 as ng
from paper_2101_10994_b200 import scenes
from oracle import nglod_oracle as O
from conftest import oracle_tree_from_golden
go = dict(np.load("/root/repo/tests/golden/octree.npz"))
svo = ng.build_octree(O.sdf_torus(0.5, 0.2), 4, go["samples_b"])
tree = oracle_tree_from_golden(go, "b_")
fld = scenes.planted_field(svo, O.sdf_torus(0.5, 0.2), seed=0, device_sdf=False)
decs = [O.OracleDecoder(d.W1, d.b1, d.W2, d.b2) for d in fld.decoders]
camd = dict(position=(0.0, 2.0, 3.5), look_at=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0), fov_y_deg=30.0, width=96, height=72)
cam = ng.Camera(**camd)
for lod in (4.0, 3.5):
    fr = O.render(tree, fld.Z, decs, camd, O.RenderParams(lod=lod, shadows=True))
    counts = []
    for k in range(6):
        fb, rep = ng.render(cam, fld, ng.RenderConfig(lod=lod, shadows=True))
        counts.append(rep.shadowed)
    print(os.environ.get("NG_FUSE_NORMALS"), lod, "oracle", int(fr.shadowed.sum()), "ours", counts,
          "color agree", float(np.mean(np.all(fb.color == fr.color, axis=-1))))
