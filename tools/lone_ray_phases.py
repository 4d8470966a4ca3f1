"""Phase clocks of the 720p frame's longest ray marched alone (NG_PROFILE
library variant, NG_LIB_VARIANT=prof): per-step microseconds of each march
phase for the one busy group (tools/march_profile.py's slots)."""
import ctypes
import os
import sys

import numpy as np

os.environ["NG_MARCH_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2101_10994_b200 as ng  # noqa: E402
from paper_2101_10994_b200 import _lib  # noqa: E402
from paper_2101_10994_b200.render import (RenderSession, device_rays, prepare_presum, resolve_config,  # noqa: E402
                                          resolve_lod)

knot, svo, fld = bench.build_workload()
cam = ng.Camera(bench.CAM["position"], bench.CAM["look_at"], bench.CAM["up"], bench.CAM["fov_y_deg"],
                bench.WIDTH, bench.HEIGHT)
config = ng.RenderConfig()
fb, rep = ng.render(cam, fld, config)
order = np.argsort(-fb.iterations.reshape(-1))
allr = cam.rays()
cfg = resolve_config(fld, config, resolve_lod(cam, fld, config))
fstruct = prepare_presum(fld, cfg)
idx = order[:1]
rays = ng.RayBundle(allr.origins[idx], allr.directions[idx])
sess = RenderSession(fld, 1, 1, n_rays=1)
d = device_rays(rays)
frame = sess.new_frame()


def step():
    _lib.call("ng_render_rays", svo.device.ref(), ctypes.byref(fstruct), ctypes.byref(cfg), _lib.ptr(d), 1,
              ctypes.byref(sess.frame_struct(frame)), ctypes.byref(sess.ws), _lib.ptr(sess.stats), 0, _lib.stream_ptr())


for _ in range(3):
    step()
torch.cuda.synchronize()
SL = 32
buf = (ctypes.c_ulonglong * (SL * 4096))()
_lib.lib().ng_march_profile(buf, 4096)
step()
torch.cuda.synchronize()
n = _lib.lib().ng_march_profile(buf, 4096)
a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, SL)[:n].astype(np.int64)
g = a[np.argmax(a[:, 0])]
MHZ = 1965.0
st = g[16]
print(f"lone ray: {int(g[0])} steps ({st} with a busy lane), span {(g[3] - g[2]) / 1e3:.1f} us, "
      f"{(g[3] - g[2]) / 1e3 / max(1, g[0]):.2f} us per step")
names = {8: "ray claims + segment walk", 9: "probe claims", 10: "flags posted", 11: "eval: voxel ids",
         12: "eval: weights/staging", 13: "eval: gather", 6: "decoder: barrier wait", 7: "decoder: GEMM + epilogue",
         15: "stop rules + publish", 18: "(eval total)", 21: "(GEMM: barrier exit to mbarrier)"}
for k, nm in names.items():
    print(f"  {nm:28s} {g[k] / max(1, st) / MHZ:.3f} us/step")
