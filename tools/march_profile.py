"""Per-group march statistics on the bench frame (NG_MARCH_PROFILE=1)."""
import ctypes, os, sys
import numpy as np
os.environ["NG_MARCH_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2101_10994_b200 as ng
from paper_2101_10994_b200 import _lib
knot, svo, fld = bench.build_workload()
cam = ng.Camera(bench.CAM["position"], bench.CAM["look_at"], bench.CAM["up"], bench.CAM["fov_y_deg"], 1280, 720)
for _ in range(3):
    fb, rep = ng.render(cam, fld, ng.RenderConfig())
buf = (ctypes.c_ulonglong * (8 * 4096))()
_lib.lib().ng_march_profile(buf, 4096)  # reset
fb, rep = ng.render(cam, fld, ng.RenderConfig())
n = _lib.lib().ng_march_profile(buf, 4096)
a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 8)[:min(n, 4096 - 1024)].astype(np.int64)
a = a[a[:, 0] > 0]
t0 = a[:, 2].min()
dur = (a[:, 3] - t0) / 1e3
steps, busy = a[:, 0], a[:, 1]
print(f"groups {len(a)}  steps total {steps.sum()}  mean {steps.mean():.1f} max {steps.max()}")
print(f"lane utilisation {busy.sum() / (steps.sum() * 128):.3f}  (trace evals {int(fb.evals.sum())})")
print(f"group end (us): min {dur.min():.0f} median {np.median(dur):.0f} p90 {np.percentile(dur, 90):.0f} max {dur.max():.0f}")
print(f"us per step (median group): {np.median(dur / steps):.2f}  acquire {np.median(a[:, 4] / steps) / 1e3:.2f}  eval {np.median(a[:, 5] / steps) / 1e3:.2f} (decoder {np.median(a[:, 7] / steps) / 1e3:.2f})")
it = fb.iterations[fb.iterations > 0]
print(f"ray iterations: mean {it.mean():.2f} p99 {np.percentile(it, 99):.0f} max {it.max()}")
order = np.argsort(dur)
for q in (0.5, 0.9, 0.99, 1.0):
    i = order[min(len(order) - 1, int(q * len(order)) - (1 if q == 1.0 else 0))]
    print(f"  q{q}: steps {steps[i]} busy/step {busy[i] / steps[i]:.1f} end {dur[i]:.0f} us")

dbg = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 8)[4096 - 1024:].astype(np.int64)
dbg = dbg[dbg[:, 0] > 0]
if len(dbg):
    tot = dbg[:, :4].sum(axis=0).astype(float)
    print("warp-0 eval phases (share): prologue %.2f staging %.2f gather %.2f decoder %.2f" % tuple(tot / tot.sum()))
