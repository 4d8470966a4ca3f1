"""Probe: per-rank frame time when a frame is split into 8-row bands over N
ranks (what each GPU of an N-GPU run renders), measured on one GPU for
every rank's band; prints the slowest and mean rank per N and the projected
speed-up (N=1 time / slowest rank), gather excluded.

    CONFIG=1|3|4 WORLDS=1,2,4,8 [BATCH=K] python tools/band_probe.py

BATCH=K renders K frames of the camera per launch (ng_render_batch) and
reports ms per frame.
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2101_10994_b200 as ng  # noqa: E402
from paper_2101_10994_b200 import _lib, scenes  # noqa: E402
from paper_2101_10994_b200.parallel import band_layout  # noqa: E402
from paper_2101_10994_b200.render import (RenderSession, camera_structs, prepare_presum, resolve_config,  # noqa: E402
                                          resolve_lod)

which = os.environ.get("CONFIG", "1")
knot, svo, fld = bench.build_workload()
if which == "1":
    W, H, config = bench.WIDTH, bench.HEIGHT, ng.RenderConfig()
else:
    _, samples = bench.knot_scene()
    svo = ng.build_octree(knot, 6, samples)
    fld = scenes.planted_field(svo, knot, seed=0)
    W, H = 1920, 1080
    config = ng.RenderConfig() if which == "3" else ng.RenderConfig(lod=4.5, shadows=True)
cam = ng.Camera(bench.CAM["position"], bench.CAM["look_at"], bench.CAM["up"], bench.CAM["fov_y_deg"], W, H)
cfg = resolve_config(fld, config, resolve_lod(cam, fld, config))
fstruct = prepare_presum(fld, cfg)
flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
out = {}
K = int(os.environ.get("BATCH", "1"))
for world in [int(w) for w in os.environ.get("WORLDS", "1,2,4,8").split(",")]:
    per_rank = []
    for rank in range(world):
        rows = len(band_layout(H, world)[rank])
        sess = RenderSession(fld, W, rows, n_rays=rows * W * K)
        fr = sess.new_frame()
        cs = camera_structs([cam.band_struct(8, world, rank)] * K)

        def step():
            _lib.call("ng_render_batch", svo.device.ref(), ctypes.byref(fstruct), ctypes.byref(cfg),
                      cs, K, ctypes.byref(sess.frame_struct(fr)), ctypes.byref(sess.ws),
                      _lib.ptr(sess.stats), _lib.stream_ptr())
        while True:
            step()
            st = sess.read_stats()
            if not sess.grow(st, cfg.trace_level + svo.device.n_virtual):
                break
        for _ in range(2):
            step()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(15)]
        for a, b in ev:
            flush.zero_()
            a.record()
            step()
            b.record()
        torch.cuda.synchronize()
        t = sorted(a.elapsed_time(b) for a, b in ev)
        per_rank.append(t[len(t) // 2] / K)
        del sess, fr
    out[world] = {"max_ms": max(per_rank), "mean_ms": sum(per_rank) / world, "ranks_ms": per_rank}
base = out[min(out)]["max_ms"]
for w, v in out.items():
    v["speedup_vs_min_world"] = base / v["max_ms"]
print(json.dumps({"config": which, "resolution": [W, H], "frames_per_launch": K, "bands": out}))
