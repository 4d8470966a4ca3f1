"""Per-frame time of frame batches (ng_render_batch) against one frame per
launch, for the last rank's bands at N = 1, 2, 4, 8 (what each GPU of an
N-GPU run renders), on one GPU; CUDA events, L2 flushed before each launch.

    CONFIG=1|3|4 KS=1,2,4,8 python tools/batch_probe.py
"""
import ctypes
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

if os.environ.get("MAX_BATCH"):  # a library variant built with -DNG_MAX_BATCH=...
    _lib.MAX_BATCH = int(os.environ["MAX_BATCH"])
which = os.environ.get("CONFIG", "1")
KS = [int(k) for k in os.environ.get("KS", "1,2,4,8").split(",")]
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
for world in [int(w) for w in os.environ.get("WORLDS", "1,2,4,8").split(",")]:
    rows = len(band_layout(H, world)[world - 1])
    base = None
    for K in KS:
        n = rows * W * K
        sess = RenderSession(fld, W, rows, n_rays=n)
        fr = sess.new_frame()
        cs = camera_structs([cam.band_struct(8, world, world - 1)] * K)

        def step():
            _lib.call("ng_render_batch", svo.device.ref(), ctypes.byref(fstruct), ctypes.byref(cfg), cs, K,
                      ctypes.byref(sess.frame_struct(fr)), ctypes.byref(sess.ws), _lib.ptr(sess.stats),
                      _lib.stream_ptr())

        while True:
            step()
            if not sess.grow(sess.read_stats(), cfg.trace_level + svo.device.n_virtual):
                break
        ms = []
        for _ in range(12):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            step()
            b.record()
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        m = sorted(ms[2:])[5] / K
        base = base or m
        print(f"config {which} N={world} (last rank, {rows} rows) K={K}: {m:.3f} ms per frame "
              f"({base / m:.2f}x K=1)", flush=True)
        del sess, fr
