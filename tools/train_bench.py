"""Time the device training epoch (configs: LOD5 knot, m=32, h=128,
500k points, batch 512) -- development probe, not the bench line."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2101_10994_b200 as ng
from paper_2101_10994_b200.trainer import DeviceTrainer

bs = int(os.environ.get("BS", 512))
npts = int(os.environ.get("NPTS", 500000))
knot, samples = bench.knot_scene()
svo = ng.build_octree(knot, 5, samples)
fld = ng.new_field(svo, seed=0)
pts = bench.query_points(knot, npts, seed=1)
dev = torch.device("cuda")
P = torch.from_numpy(pts).to(dev)
D = knot.device_eval(P)
tr = DeviceTrainer(ng.NeuralField(svo, fld.Z.astype(np.float64), [d.astype(np.float64) for d in fld.decoders]), bs)
act = [1, 2, 3, 4, 5]
tr.run_epoch(P, D, act, True, 1e-3)  # warm
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
times = []
for k in range(3):
    e0.record(); tr.run_epoch(P, D, act, True, 1e-3); e1.record(); torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
sums = tr.level_sums.cpu().numpy() / npts
print(json.dumps({"batch": bs, "points": npts, "epoch_ms": times, "Mpts_per_s": npts / (min(times) * 1e3),
                  "us_per_batch": min(times) * 1e3 / ((npts + bs - 1) // bs), "losses": sums.tolist(),
                  "status": int(tr.status.item()), "corners": svo.corner_count}))
if os.environ.get("NG_TRAIN_EVENTS") == "1":
    import ctypes
    from paper_2101_10994_b200 import _lib
    buf = (ctypes.c_double * 6)()
    _lib.lib().ng_train_profile(buf)
    names = ["locate", "rowprep", "gather", "dec", "reduce", "update"]
    print(json.dumps({k: round(buf[i] * 1e3, 2) for i, k in enumerate(names)}), "us per batch (events, synced)")
