"""Per-group march statistics (NG_MARCH_PROFILE=1 with the NG_PROFILE
library variant: tools/build_variant.sh prof "-DNG_PROFILE"; run with
NG_LIB_VARIANT=prof).

    CONFIG=1|3|4 [BAND=world,rank] [BATCH=K] python tools/march_profile.py

Prints the groups' step counts, lane utilisation, the spread of group end
times, the time per step split into acquire / eval / decoder, the ray
iteration distribution and, for the slowest groups, steps vs end time (the
tail: its us/step is the per-step latency at light load).
"""
import ctypes
import os
import sys

import numpy as np

os.environ["NG_MARCH_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2101_10994_b200 as ng  # noqa: E402
from paper_2101_10994_b200 import _lib, scenes  # noqa: E402
from paper_2101_10994_b200.parallel import band_layout  # noqa: E402
from paper_2101_10994_b200.render import (RenderSession, camera_structs, prepare_presum, resolve_config,  # noqa: E402
                                          resolve_lod)

which = os.environ.get("CONFIG", "1")
band = os.environ.get("BAND")
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
world, rank = (int(v) for v in band.split(",")) if band else (1, 0)
rows = len(band_layout(H, world)[rank])
K = int(os.environ.get("BATCH", "1"))
sess = RenderSession(fld, W, rows, n_rays=rows * W * K)
fr = sess.new_frame()
cs = camera_structs([cam.band_struct(8, world, rank)] * K)


def step():
    _lib.call("ng_render_batch", svo.device.ref(), ctypes.byref(fstruct), ctypes.byref(cfg), cs, K,
              ctypes.byref(sess.frame_struct(fr)), ctypes.byref(sess.ws), _lib.ptr(sess.stats), _lib.stream_ptr())


while True:
    step()
    if not sess.grow(sess.read_stats(), cfg.trace_level + svo.device.n_virtual):
        break
for _ in range(3):
    step()
torch.cuda.synchronize()
SL = 32  # NG_PROF_SLOTS
buf = (ctypes.c_ulonglong * (SL * 4096))()
_lib.lib().ng_march_profile(buf, 4096)  # reset
has_tl = hasattr(_lib.lib(), "ng_march_timeline")
if has_tl:
    _lib.lib().ng_march_timeline(None)  # allocate / reset the step timeline
a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a0.record()
step()
b0.record()
torch.cuda.synchronize()
n = _lib.lib().ng_march_profile(buf, 4096)
tl = None
if has_tl:
    tbuf = (ctypes.c_ulonglong * (64 * 512))()
    _lib.lib().ng_march_timeline(tbuf)
    tl = np.frombuffer(tbuf, dtype=np.uint64).reshape(64, 512)
a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, SL)[:n].astype(np.int64)
a = a[a[:, 0] > 0]
t0 = a[:, 2].min()
dur = (a[:, 3] - t0) / 1e3
steps, busy = a[:, 0], a[:, 1]
print(f"config {which} band {world},{rank}: frame {a0.elapsed_time(b0):.3f} ms (profiled build)")
print(f"groups {len(a)}  steps total {steps.sum()}  mean {steps.mean():.1f} max {steps.max()}")
print(f"lane utilisation {busy.sum() / (steps.sum() * 128):.3f}")
print(f"group end (us): min {dur.min():.0f} median {np.median(dur):.0f} p90 {np.percentile(dur, 90):.0f} "
      f"max {dur.max():.0f}")
print(f"us per step (median group): {np.median(dur / steps):.2f}")
order = np.argsort(dur)
for q in (0.5, 0.9, 0.99, 1.0):
    i = order[min(len(order) - 1, int(q * len(order)) - (1 if q == 1.0 else 0))]
    print(f"  q{q}: steps {steps[i]} busy/step {busy[i] / steps[i]:.1f} end {dur[i]:.0f} us")
# light-load steps: the slowest 5 groups' last steps are mostly 1-4 lanes
slow = order[-5:]
print("slowest groups: steps", steps[slow].tolist(), "busy/step", np.round(busy[slow] / steps[slow], 1).tolist())
# group-leader clock64 phases per step (cycles -> us at the SM clock)
MHZ = float(os.environ.get("SM_MHZ", "1965"))
names = {8: "ray claims + segment walk", 9: "probe claims", 10: "group barrier", 11: "eval: voxel ids",
         12: "eval: weights/staging", 13: "eval: gather", 6: "decoder: barrier wait", 7: "decoder: GEMM + epilogue",
         15: "stop rules + publish"}
st = a[:, 16].sum()
print(f"phase us per group step (all groups, {st} steps):")
for k, nm in names.items():
    print(f"  {nm:28s} {a[:, k].sum() / st / MHZ:.3f}")
print(f"  {'eval total (slot 18)':28s} {a[:, 18].sum() / st / MHZ:.3f}")
light = a[:, 17].sum()
if light:
    print(f"light steps (<= 8 busy lanes): {light}, us per light step {a[:, 19].sum() / light / MHZ:.2f}")
i = order[-1]
print("slowest group phases (us/step):", {names[k]: round(a[i, k] / a[i, 16] / MHZ, 3) for k in names})
# busy lanes per group step over the march's time (64 sampled groups, 10 time bins)
if tl is not None:
    ts = (tl >> 8).astype(np.int64)
    act = (tl & 0xff).astype(np.int64)
    valid = ts > 0
    if valid.any():
        t0l, t1l = ts[valid].min(), ts[valid].max()
        bins = np.minimum(((ts - t0l) * 10 // max(1, t1l - t0l + 1)), 9)
        row = []
        for bi in range(10):
            sel = valid & (bins == bi)
            row.append(f"{act[sel].mean():.0f}/{sel.sum()}" if sel.any() else "-")
        print(f"timeline (64 groups; mean busy lanes per step / steps, per tenth of {(t1l - t0l) / 1e3:.0f} us):",
              " ".join(row))
# the frame's ray iteration distribution via the public API (non-profiled timing irrelevant here)
if world == 1 and K == 1:
    fb, rep = ng.render(cam, fld, config)
    itr = fb.iterations[fb.iterations > 0]
    print(f"ray iterations: n {itr.size} mean {itr.mean():.2f} p99 {np.percentile(itr, 99):.0f} "
          f"p99.9 {np.percentile(itr, 99.9):.0f} max {itr.max()}  (>=100: {(itr >= 100).sum()})")
