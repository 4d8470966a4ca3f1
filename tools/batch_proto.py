"""Prototype: K frames of one camera stacked in one launch pair (variant
built with -DNG_BATCH_PROTO=K), time per frame vs one frame per launch."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2101_10994_b200 as ng  # noqa: E402
from paper_2101_10994_b200 import _lib, scenes  # noqa: E402
from paper_2101_10994_b200.parallel import band_layout  # noqa: E402
from paper_2101_10994_b200.render import RenderSession, prepare_presum, resolve_config, resolve_lod  # noqa: E402

K = int(os.environ.get("K", "1"))
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
for world in (1, 2, 4, 8):
    rows = len(band_layout(H, world)[world - 1])
    n = rows * W * K
    sess = RenderSession(fld, W, rows * K, n_rays=n)
    fr = sess.new_frame()
    cs = cam.band_struct(8, world, world - 1)
    cs.local_rows = rows * K

    def step():
        _lib.call("ng_render_frame", svo.device.ref(), ctypes.byref(fstruct), ctypes.byref(cfg), ctypes.byref(cs),
                  ctypes.byref(sess.frame_struct(fr)), ctypes.byref(sess.ws), _lib.ptr(sess.stats), _lib.stream_ptr())

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
    m = sorted(ms[2:])[5]
    hits = int(fr["hit"].sum().item())
    print(f"config {which} world {world} (last band, {rows} rows) K={K}: launch {m:.3f} ms, per frame {m / K:.3f} ms,"
          f" hits/frame {hits / K:.0f}", flush=True)
