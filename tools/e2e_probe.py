"""Where the end-to-end render() time goes (wall clock, 720p knot frame)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2101_10994_b200 as ng
import importlib
R = importlib.import_module("paper_2101_10994_b200.render")
knot, svo, fld = bench.build_workload()
cam = ng.Camera(bench.CAM["position"], bench.CAM["look_at"], bench.CAM["up"], bench.CAM["fov_y_deg"], 1280, 720)
config = ng.RenderConfig()
for _ in range(3):
    fb, rep = ng.render(cam, fld, config); _ = fb.color
torch.cuda.synchronize()

def wall(f, n=30):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3

lod = R.resolve_lod(cam, fld, config); cfg = R.resolve_config(fld, config, lod)
sess = R._session(fld, 1280, 720)
frame = sess.new_frame()
print("enqueue only (device bound)", wall(lambda: sess.enqueue(cfg, frame, camera=cam)))
print("enqueue + stats sync", wall(lambda: (sess.enqueue(cfg, frame, camera=cam), sess.read_stats())))
def with_color():
    sess.enqueue(cfg, frame, camera=cam)
    h = torch.empty(frame["color"].shape, dtype=torch.uint8, pin_memory=True)
    h.copy_(frame["color"], non_blocking=True)
    sess.read_stats()
print("enqueue + color D2H + stats", wall(with_color))
print("new_frame", wall(lambda: sess.new_frame(), 200))
print("resolve", wall(lambda: (R.resolve_lod(cam, fld, config), R.resolve_config(fld, config, lod)), 200))
print("render()", wall(lambda: ng.render(cam, fld, config)))
print("render() + color", wall(lambda: ng.render(cam, fld, config)[0].color))

# host-side cost of one enqueue (no sync), and its parts
def host(f, n=200):
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    dt = (time.perf_counter() - t0) / n * 1e3
    torch.cuda.synchronize()
    return dt
print("host: enqueue", host(lambda: sess.enqueue(cfg, frame, camera=cam), 50))
print("host: camera.struct", host(lambda: cam.struct()))
print("host: prepare_presum", host(lambda: R.prepare_presum(fld, cfg)))
print("host: frame_struct", host(lambda: sess.frame_struct(frame)))
fs = sess.frame_struct(frame); cs = cam.struct()
import ctypes
from paper_2101_10994_b200._lib import call, ptr, stream_ptr
print("host: call only", host(lambda: call("ng_render_frame", fld.svo.device.ref(), fld.device.ref(), ctypes.byref(cfg),
      ctypes.byref(cs), ctypes.byref(fs), ctypes.byref(sess.ws), ptr(sess.stats), stream_ptr()), 50))
print("host: refs", host(lambda: (fld.svo.device.ref(), fld.device.ref(), stream_ptr())))
