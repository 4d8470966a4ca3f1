"""Frame time of configs[1] (720p LOD5), configs[3] (1080p LOD6) and
configs[4] (1080p LOD4.5 + shadows) through TiledRenderer at N=1, CUDA
events, L2 flushed, median of 10 (the bench's timing)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2101_10994_b200 as ng
from paper_2101_10994_b200 import scenes
from paper_2101_10994_b200.parallel import TiledRenderer
from paper_2101_10994_b200.render import resolve_config, resolve_lod
knot, svo, fld = bench.build_workload()
flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
which = os.environ.get("CFGS", "1,3,4").split(",")
out = {}
class A: steps = 10
if "1" in which:
    cam = ng.Camera(bench.CAM["position"], bench.CAM["look_at"], bench.CAM["up"], bench.CAM["fov_y_deg"], 1280, 720)
    t = TiledRenderer(fld, 1280, 720)
    t.render(cam, ng.RenderConfig())
    cfg = resolve_config(fld, ng.RenderConfig(), resolve_lod(cam, fld, ng.RenderConfig()))
    out["c1"] = bench._time_tiled(t, cam, cfg, 10, flush, 1)
if "3" in which or "4" in which:
    _, samples = bench.knot_scene()
    svo6 = ng.build_octree(knot, 6, samples)
    fld6 = scenes.planted_field(svo6, knot, seed=0)
    cam = ng.Camera(bench.CAM["position"], bench.CAM["look_at"], bench.CAM["up"], bench.CAM["fov_y_deg"], 1920, 1080)
    for k, config in (("c3", ng.RenderConfig()), ("c4", ng.RenderConfig(lod=4.5, shadows=True))):
        if k[1] not in which:
            continue
        t = TiledRenderer(fld6, 1920, 1080)
        t.render(cam, config)
        cfg = resolve_config(fld6, config, resolve_lod(cam, fld6, config))
        out[k] = bench._time_tiled(t, cam, cfg, 10, flush, 1)
print(json.dumps(out))
