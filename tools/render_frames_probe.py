"""render_frames (double-buffered readback) vs render() frames/s on the 720p
knot frame, end to end with the colour image on the host."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_2101_10994_b200 as ng, importlib
R = importlib.import_module("paper_2101_10994_b200.render")
knot, svo, fld = bench.build_workload()
cam = ng.Camera(bench.CAM["position"], bench.CAM["look_at"], bench.CAM["up"], bench.CAM["fov_y_deg"], 1280, 720)
cfg = ng.RenderConfig()
for trial in range(3):
    for fb, r in ng.render_frames([cam] * 8, fld, cfg):
        _ = fb.color
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for fb, r in ng.render_frames([cam] * 40, fld, cfg):
        img = fb.color
    dt = (time.perf_counter() - t0) / 40
    sess = R._session(fld, 1280, 720)
    print(f"render_frames {1/dt:.0f} fps; graphs {len(sess._graphs)} replays {sess.graph_replays} misses {sess._graph_misses}")
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(40):
    fb, r = ng.render(cam, fld, cfg); img = fb.color
print(f"render {40/(time.perf_counter()-t0):.0f} fps")
