"""Subprocess helper for tests/test_gpu_tile_traverse.py: renders the
golden planted-torus frame with whatever NG_TILE_* / NG_TILE_TRAVERSE knobs
the environment sets (they are read once per process) and saves the frame.

    python tests/tile_probe.py OUT.npz [tiny_pairs]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import importlib  # noqa: E402

import paper_2101_10994_b200 as ng  # noqa: E402
from paper_2101_10994_b200 import scenes  # noqa: E402

R = importlib.import_module("paper_2101_10994_b200.render")  # the module (the package exports render())
from oracle import nglod_oracle as O  # noqa: E402

out = sys.argv[1]
grows = [0]
if len(sys.argv) > 2 and sys.argv[2] == "tiny_pairs":
    # start from a workspace far too small, so the tile lists overflow the
    # arena and the frame reruns after growing (render.py's grow loop)
    init0, grow0 = R.RenderSession.__init__, R.RenderSession.grow

    def init(self, *a, **k):
        init0(self, *a, **k)
        self.pair_cap = 64
        self._alloc_ws()

    def grow(self, st, n_levels):
        again = grow0(self, st, n_levels)
        grows[0] += int(again)
        return again
    R.RenderSession.__init__, R.RenderSession.grow = init, grow

go = dict(np.load(os.path.join(ROOT, "tests", "golden", "octree.npz")))
svo = ng.build_octree(O.sdf_torus(0.5, 0.2), 4, go["samples_b"])
fld = scenes.planted_field(svo, O.sdf_torus(0.5, 0.2), seed=0, device_sdf=False)
cam = ng.Camera((0.0, 2.0, 3.5), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 30.0, 96, 72)
fb, rep = ng.render(cam, fld, ng.RenderConfig())
# the frame's final (ray, voxel, t_enter, t_exit) lists, in the reference's order
sess = R._session(fld, cam.width, cam.height)
fin = sess.final_list(svo.max_level)
# tile traversal continuations pushed by the last frame (traverse.cu: split tiles)
import ctypes  # noqa: E402
from paper_2101_10994_b200 import _lib  # noqa: E402
off = (ctypes.c_int64 * 5)()
_lib.check(_lib.lib().ng_render_workspace_offsets(sess.n, sess.pair_cap, sess.hit_cap, off, 5), "offsets")
splits = int(sess.ws_buf[off[4] + 128:off[4] + 136].view(torch.int64).item()) >> 32
np.savez(out, hit=fb.hit, t=fb.t, color=fb.color, iterations=fb.iterations, evals=fb.evals, normal=fb.normal,
         normal_ok=fb.normal_ok,
         visible=rep.visible, n_evals=rep.evals, grows=grows[0],
         l_rays=fin.rays, l_voxels=fin.voxels, l_t_enter=fin.t_enter, l_t_exit=fin.t_exit, splits=splits)
