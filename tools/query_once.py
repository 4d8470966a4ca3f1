"""One configs[2] batched query (forward L=1..5, 2^24 points) after a
warm-up call; run under ncu to capture k_query_tc:

    ncu --set full -k regex:k_query_tc -s 1 -c 1 -o gpurun_out/query python tools/query_once.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2101_10994_b200.field import forward_levels_device  # noqa: E402

knot, svo, fld = bench.build_workload()
pts = torch.from_numpy(bench.query_points(knot, bench.QUERY_POINTS)).to("cuda")
for _ in range(2):
    out = forward_levels_device(svo, fld.device, pts, [1, 2, 3, 4, 5])
torch.cuda.synchronize()
print("query ok", out.shape)
