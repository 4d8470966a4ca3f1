"""The configs[2] query timed two ways in one process: through
forward_levels_device (output and counters allocated per call) and through
ng_query on preallocated buffers; per-call ms, L2 write-flushed before each."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2101_10994_b200 import _lib  # noqa: E402
from paper_2101_10994_b200.field import _Counters, forward_levels_device  # noqa: E402

knot, svo, fld = bench.build_workload()
dev = torch.device("cuda:0")
pts = torch.from_numpy(bench.query_points(knot, bench.QUERY_POINTS)).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
n = pts.shape[0]
out = torch.empty((n, 5), dtype=torch.float64, device=dev)
cnt = _Counters()
args = _lib.NgQueryArgs(0b11111, -1, 0, 0, 0.0)


def direct():
    _lib.call("ng_query", svo.device.ref(), fld.device.ref(), ctypes.byref(args), _lib.ptr(pts), n, _lib.ptr(out),
              cnt.ptr(), _lib.stream_ptr())


def api():
    return forward_levels_device(svo, fld.device, pts, [1, 2, 3, 4, 5])


for f in (direct, api, direct):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    ms = []
    for _ in range(9):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = f()
        b.record()
        torch.cuda.synchronize()
        ms.append(round(a.elapsed_time(b), 2))
        del r
    print(f.__name__, "median", sorted(ms)[4], "calls", ms)
