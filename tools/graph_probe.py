"""Probe: frame time with plain launches vs one captured CUDA graph replay."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2101_10994_b200 as ng
from paper_2101_10994_b200.render import RenderSession, resolve_config, resolve_lod

knot, svo, fld = bench.build_workload()
cam = ng.Camera(bench.CAM["position"], bench.CAM["look_at"], bench.CAM["up"], bench.CAM["fov_y_deg"], bench.WIDTH, bench.HEIGHT)
config = ng.RenderConfig()
cfg = resolve_config(fld, config, resolve_lod(cam, fld, config))
sess = RenderSession(fld, bench.WIDTH, bench.HEIGHT)
fr = sess.new_frame()
for _ in range(3):
    sess.enqueue(cfg, fr, camera=cam)
st = sess.read_stats(); assert not st.overflow
flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

def timeit(fn, k=50, do_flush=True):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for a, b in ev:
        if do_flush: flush.zero_()
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    return t[len(t) // 2]

plain = timeit(lambda: sess.enqueue(cfg, fr, camera=cam))
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    sess.enqueue(cfg, fr, camera=cam)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        sess.enqueue(cfg, fr, camera=cam)
torch.cuda.synchronize()
graph = timeit(lambda: g.replay())
st2 = sess.read_stats()
print(json.dumps({"plain_ms": plain, "graph_ms": graph, "plain_noflush": timeit(lambda: sess.enqueue(cfg, fr, camera=cam), do_flush=False),
                  "graph_noflush": timeit(lambda: g.replay(), do_flush=False), "visible": int(st2.visible)}))
