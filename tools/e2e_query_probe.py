"""Where the end-to-end configs[2] query time goes (numpy in, numpy out)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2101_10994_b200.field import forward_levels_device  # noqa: E402

knot, svo, fld = bench.build_workload()
pts_h = np.ascontiguousarray(bench.query_points(knot, bench.QUERY_POINTS))
dev = torch.device("cuda", 0)
L = bench.QUERY_LEVELS


def wall(f, n=3):
    out = []
    for _ in range(n + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        out.append((time.perf_counter() - t0) * 1e3)
    return sorted(out[1:])[len(out[1:]) // 2], r


print("thp:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip() if os.path.exists(
    "/sys/kernel/mm/transparent_hugepage/enabled") else "n/a", " cpus:", os.cpu_count())
ms, _ = wall(lambda: bool(np.any(pts_h < -1.0) or np.any(pts_h > 1.0)))
print(f"domain check (numpy) {ms:.1f} ms")
ms, d = wall(lambda: torch.from_numpy(pts_h).to(dev))
print(f"H2D pageable {ms:.1f} ms ({pts_h.nbytes / ms / 1e6:.1f} GB/s)")
pin = torch.empty(pts_h.shape, dtype=torch.float64, pin_memory=True)
ms, _ = wall(lambda: pin.numpy().__setitem__(slice(None), pts_h))
print(f"numpy -> pinned memcpy {ms:.1f} ms")
ms, _ = wall(lambda: d.copy_(pin, non_blocking=True))
print(f"H2D pinned {ms:.1f} ms ({pts_h.nbytes / ms / 1e6:.1f} GB/s)")
ms, out = wall(lambda: forward_levels_device(svo, fld.device, d, L))
print(f"query kernel {ms:.1f} ms")
ms, h = wall(lambda: out.cpu())
print(f"D2H pageable .cpu() {ms:.1f} ms ({out.numel() * 8 / ms / 1e6:.1f} GB/s)")
pout = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
ms, _ = wall(lambda: pout.copy_(out, non_blocking=True))
print(f"D2H pinned {ms:.1f} ms ({out.numel() * 8 / ms / 1e6:.1f} GB/s)")
ms, a = wall(lambda: np.empty(tuple(out.shape)))
print(f"np.empty {ms:.1f} ms")
ms, _ = wall(lambda: np.copyto(np.empty(tuple(out.shape)), pout.numpy()))
print(f"pinned -> fresh numpy copy (first touch) {ms:.1f} ms")
dst = np.empty(tuple(out.shape))
dst[:] = 0
ms, _ = wall(lambda: np.copyto(dst, pout.numpy()))
print(f"pinned -> touched numpy copy {ms:.1f} ms")
ms, r = wall(lambda: fld.forward_levels(pts_h, L))
print(f"public forward_levels {ms:.1f} ms -> {len(pts_h) / ms / 1e3:.1f} Mpoints/s")
