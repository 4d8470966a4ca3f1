"""Query-leg variance between processes: best-of-7 Mpoints/s of the bench's
configs[2] query, with the addresses of the field's tables (run it several
times, one process each)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2101_10994_b200.field import forward_levels_device
knot, svo, fld = bench.build_workload()
dev = torch.device("cuda:0")
pts = torch.from_numpy(bench.query_points(knot, bench.QUERY_POINTS)).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(2):
    out = forward_levels_device(svo, fld.device, pts, [1, 2, 3, 4, 5])
torch.cuda.synchronize()
ms = []
mode = os.environ.get("QP_FLUSH", "write")  # write (as bench.py) | read | none
acc = torch.zeros((), dtype=torch.int64, device=dev)
for _ in range(7):
    if mode == "write":
        flush.zero_()
    elif mode == "read":
        acc += flush.view(torch.int64).max()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    forward_levels_device(svo, fld.device, pts, [1, 2, 3, 4, 5], out=out)  # resident output
    b.record()
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
z = fld.device.Z
print(f"flush {mode}  best {bench.QUERY_POINTS / min(ms) / 1e3:.0f} Mpts/s  median {bench.QUERY_POINTS / sorted(ms)[3] / 1e3:.0f}"
      f"  Z {z.data_ptr():#x} ({z.numel() * 4 >> 20} MiB)  pts {pts.data_ptr():#x}  out {out.data_ptr():#x}"
      f"  calls ms {[round(v, 2) for v in ms]}")
