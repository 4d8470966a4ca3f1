"""Wall time per frame of render_frames(batch=K) at configs[1] (colour
image read back per frame), with the session's graph replays and misses."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2101_10994_b200 as ng  # noqa: E402
R = sys.modules["paper_2101_10994_b200.render"]

knot, svo, fld = bench.build_workload()
cam = ng.Camera(bench.CAM["position"], bench.CAM["look_at"], bench.CAM["up"], bench.CAM["fov_y_deg"],
                bench.WIDTH, bench.HEIGHT)
cfg = ng.RenderConfig()
for K in [int(k) for k in os.environ.get("KS", "8,16").split(",")]:
    n = 2 * K
    for _ in range(2):
        for fb, _r in ng.render_frames([cam] * n, fld, cfg, batch=K):
            _ = fb.color
    torch.cuda.synchronize()
    sess = R._session(fld, bench.WIDTH, bench.HEIGHT, K)
    m0, r0 = sess._graph_misses, sess.graph_replays
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        for fb, rep in ng.render_frames([cam] * n, fld, cfg, batch=K):
            img = fb.color
        ts.append((time.perf_counter() - t0) / n)
    print(f"K={K}: {1e3 * min(ts):.3f} / {1e3 * sorted(ts)[1]:.3f} ms per frame (best / median of 3 runs of {n}), "
          f"graph replays {sess.graph_replays - r0}, misses now {sess._graph_misses} (was {m0}), "
          f"graphs {len(sess._graphs)}", flush=True)

if os.environ.get("PROFILE"):
    import cProfile
    import pstats
    K = int(os.environ["PROFILE"])
    pr = cProfile.Profile()
    pr.enable()
    for fb, rep in ng.render_frames([cam] * (2 * K), fld, cfg, batch=K):
        img = fb.color
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
