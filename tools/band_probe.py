"""Probe: per-rank frame time when the 720p frame is split into 8-row bands
over N ranks (what each GPU of an N-GPU run renders), on one GPU."""
import os, sys, json, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2101_10994_b200 as ng
from paper_2101_10994_b200 import _lib
from paper_2101_10994_b200.parallel import band_layout
from paper_2101_10994_b200.render import RenderSession, prepare_presum, resolve_config, resolve_lod

knot, svo, fld = bench.build_workload()
W, H = bench.WIDTH, bench.HEIGHT
cam = ng.Camera(bench.CAM["position"], bench.CAM["look_at"], bench.CAM["up"], bench.CAM["fov_y_deg"], W, H)
cfg = resolve_config(fld, ng.RenderConfig(), resolve_lod(cam, fld, ng.RenderConfig()))
prepare_presum(fld, cfg)
flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
out = {}
for world in [int(w) for w in os.environ.get("WORLDS", "1,2,4,8").split(",")]:
    rows = len(band_layout(H, world)[0])
    sess = RenderSession(fld, W, rows, n_rays=rows * W)
    fr = sess.new_frame()
    cs = cam.band_struct(8, world, 0)
    def step():
        _lib.call("ng_render_frame", svo.device.ref(), fld.device.ref(), ctypes.byref(cfg), ctypes.byref(cs),
                  ctypes.byref(sess.frame_struct(fr)), ctypes.byref(sess.ws), _lib.ptr(sess.stats), _lib.stream_ptr())
    for _ in range(3):
        step()
    st = sess.read_stats(); assert not st.overflow
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for a, b in ev:
        flush.zero_(); a.record(); step(); b.record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    out[world] = {"ms": t[len(t) // 2], "rows": rows, "visible": int(st.visible)}
print(json.dumps(out))
