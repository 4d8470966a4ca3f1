"""Per-step latency of a ray marched alone: the configs[1] frame's longest
rays (most sphere-tracing iterations), each set traced by itself through
ng_render_rays (traversal + march, no normals), timed with CUDA events;
frame time / iterations is the lone-ray step latency that bounds an N-GPU
band's tail."""
import ctypes
import os
import sys

import numpy as np

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
it = fb.iterations.reshape(-1)
order = np.argsort(-it)
allr = cam.rays()
cfg = resolve_config(fld, config, resolve_lod(cam, fld, config))
fstruct = prepare_presum(fld, cfg)
for k in (1, 8, 64):
    idx = order[:k]
    rays = ng.RayBundle(allr.origins[idx], allr.directions[idx])
    sess = RenderSession(fld, k, 1, n_rays=k)
    d = device_rays(rays)
    frame = sess.new_frame()

    def step():
        _lib.call("ng_render_rays", svo.device.ref(), ctypes.byref(fstruct), ctypes.byref(cfg), _lib.ptr(d), k,
                  ctypes.byref(sess.frame_struct(frame)), ctypes.byref(sess.ws), _lib.ptr(sess.stats), 0,
                  _lib.stream_ptr())
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ms = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    m = sorted(ms)[5]
    iters = int(frame["iterations"][:k].max().item())
    print(f"{k:3d} longest rays alone: frame {m * 1e3:.1f} us, max iterations {iters} "
          f"(in the frame {it[idx].max()}), {m * 1e3 / max(iters, 1):.2f} us per step")
