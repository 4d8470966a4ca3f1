"""Per-tile timing of k_traverse_tiles (NG_PROFILE library variant:
tools/build_variant.sh prof "-DNG_PROFILE"; run with NG_LIB_VARIANT=prof).

    CONFIG=1|3 [BAND=world,rank] python tools/tile_profile.py

Prints the kernel span, the tile duration distribution, the slowest tiles
(duration, final pairs, start offset) and how much of the span the slowest
tile's warp alone accounts for (the straggler tail)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2101_10994_b200 as ng  # noqa: E402
from paper_2101_10994_b200 import _lib, scenes  # noqa: E402
from paper_2101_10994_b200.parallel import band_layout  # noqa: E402
from paper_2101_10994_b200.render import RenderSession, prepare_presum, resolve_config, resolve_lod  # noqa: E402

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
    config = ng.RenderConfig()
cam = ng.Camera(bench.CAM["position"], bench.CAM["look_at"], bench.CAM["up"], bench.CAM["fov_y_deg"], W, H)
cfg = resolve_config(fld, config, resolve_lod(cam, fld, config))
fstruct = prepare_presum(fld, cfg)
world, rank = (int(v) for v in band.split(",")) if band else (1, 0)
rows = len(band_layout(H, world)[rank])
n = rows * W
sess = RenderSession(fld, W, rows, n_rays=n)
fr = sess.new_frame()
cs = cam.band_struct(8, world, rank)
lib = _lib.lib()
n_tiles = (n + 31) // 32
assert lib.ng_tile_profile_enable(ctypes.c_longlong(n_tiles)) == 0


def step():
    _lib.call("ng_render_frame", svo.device.ref(), ctypes.byref(fstruct), ctypes.byref(cfg), ctypes.byref(cs),
              ctypes.byref(sess.frame_struct(fr)), ctypes.byref(sess.ws), _lib.ptr(sess.stats), _lib.stream_ptr())


while True:
    step()
    if not sess.grow(sess.read_stats(), cfg.trace_level + svo.device.n_virtual):
        break
for _ in range(3):
    step()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (4 * n_tiles))()
lib.ng_tile_profile_read(buf, ctypes.c_longlong(n_tiles))  # reset
step()
torch.cuda.synchronize()
lib.ng_tile_profile_read(buf, ctypes.c_longlong(n_tiles))
a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 4).astype(np.int64)
t0 = a[:, 0].min()
start = (a[:, 0] - t0) / 1e3
dur = (a[:, 1] - a[:, 0]) / 1e3
end = start + dur
print(f"config {which} band {world},{rank}: {n_tiles} tiles, span {end.max():.1f} us, "
      f"sum of tile time {dur.sum():.0f} us over {len(np.unique(a[:, 3]))} warps")
print(f"tile us: median {np.median(dur):.2f} p90 {np.percentile(dur, 90):.2f} p99 {np.percentile(dur, 99):.2f} "
      f"max {dur.max():.1f}")
order = np.argsort(-dur)
for i in order[:8]:
    print(f"  tile {i}: {dur[i]:.1f} us, final pairs {a[i, 2]}, start {start[i]:.1f} us, end {end[i]:.1f} us")
w_end = {}
for i in range(n_tiles):
    w_end[a[i, 3]] = max(w_end.get(a[i, 3], 0.0), end[i])
we = np.array(list(w_end.values()))
print(f"warp end us: median {np.median(we):.1f} p90 {np.percentile(we, 90):.1f} max {we.max():.1f}")
print(f"pairs vs time: corr {np.corrcoef(a[:, 2], dur)[0, 1]:.3f}; us per 100 final pairs (heavy tiles) "
      f"{np.median(dur[a[:, 2] > 500] / a[a[:, 2] > 500, 2] * 100) if (a[:, 2] > 500).any() else 0:.2f}")
# per-part records (continuations included): NG_PROFILE builds with ng_part_profile
if hasattr(lib, "ng_part_profile"):
    lib.ng_part_profile(None, 1)
    step()
    torch.cuda.synchronize()
    pb = (ctypes.c_ulonglong * (8 << 20))()
    k = lib.ng_part_profile(pb, 1)
    p = np.frombuffer(pb, dtype=np.uint64)[:8 * k].reshape(-1, 8).astype(np.int64)
    if k:
        t0p = p[:, 0].min()
        pdur = (p[:, 1] - p[:, 0]) / 1e3
        cont = p[:, 2] >= 0
        print(f"parts {k}: fresh {int((~cont).sum())}, continuations {int(cont.sum())}, splits {int(p[:, 6].sum())}, "
              f"split time {p[:, 7].sum() / 1e3:.0f} us total")
        for nm, sel in (("fresh", ~cont), ("cont", cont)):
            if sel.any():
                d = pdur[sel]
                print(f"  {nm}: median {np.median(d):.1f} p99 {np.percentile(d, 99):.1f} max {d.max():.1f} us; "
                      f"split us in the slowest: {p[sel][np.argmax(d), 7] / 1e3:.1f} ({p[sel][np.argmax(d), 6]} splits)")
        o = np.argsort(-pdur)[:6]
        for i in o:
            print(f"   part rec {p[i, 2]} tile {p[i, 3]} t0 {p[i, 4]} start {(p[i, 0] - t0p) / 1e3:.1f} "
                  f"dur {pdur[i]:.1f} splits {p[i, 6]} split_us {p[i, 7] / 1e3:.1f}")
