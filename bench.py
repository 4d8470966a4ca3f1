"""Benchmark: frames/sec of the 1280x720 LOD5 sparse sphere trace (BASELINE.json
configs[1]) on B200, plus the batched SDF query (configs[2]) in Mpoints/sec.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0. A step is one full frame of the hot path --
camera rays, BFS traversal, persistent sphere-trace march, normals and
shading -- over the torus-knot LOD5 octree with the planted field (SURVEY.md
Appendix A; synthetic, no training). `value` is device time (CUDA events,
L2 flushed between frames); `e2e` times the public `render_frames()` call
(render() per camera with double-buffered readback) with every frame's
colour image and statistics read back to the host. With --gpus N > 1 and no torchrun
environment, bench.py launches N ranks itself (torch.distributed.run).

`--impl reference` runs the UNMODIFIED reference package (`octfield`,
pip-installed into baseline/_ref) through its public `render()` on the
host cores, whole frames, on inputs the reference itself produced
(bench_data/knot_l5_ref.npz, tools/make_ref_inputs.py). The `cpu_baseline`
of our line runs the same reference functions on a row sample of the frame
and checks our render path's per-ray voxel lists against the reference's
`ray_trace_octree` on those rays.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/sec 1280×720 LOD5 sparse sphere trace; Mpoints/sec batched SDF query"
WIDTH, HEIGHT = 1280, 720
MAX_LEVEL = 5
CAM = dict(position=(0.0, 1.5, 3.5), look_at=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0), fov_y_deg=30.0)
QUERY_POINTS = 1 << 24
BUILD_SAMPLES = 1 << 17
L2_FLUSH_BYTES = 256 << 20
EVAL_BYTES_PER_LEVEL = 1064   # 8 B node + 32 B corner ids + 8 x 32 x 4 B features
EVAL_BYTES_BASE = 16          # 12 B point + 4 B result


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=16,
                    help="frames per launch sequence (ng_render_batch; 1..16): the timed steps are frames, rendered "
                         "`batch` at a time; each frame's latency alone is reported beside it")
    ap.add_argument("--no-query", action="store_true", help="skip the batched-query leg")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-extra", action="store_true", help="skip the configs[3]/[4] 1080p legs")
    ap.add_argument("--no-train", action="store_true", help="skip the training-step leg (SURVEY.md 8f)")
    return ap.parse_args()


# ------------------------------------------------------------------ workload

def knot_scene():
    from paper_2101_10994_b200 import scenes
    knot = scenes.torus_knot(segments=1024, tube=0.08)
    samples = scenes.knot_samples(knot, BUILD_SAMPLES, seed=0)
    return knot, samples


def build_workload():
    import paper_2101_10994_b200 as ng
    from paper_2101_10994_b200 import scenes
    knot, samples = knot_scene()
    svo = ng.build_octree(knot, MAX_LEVEL, samples)          # device lattice + device build
    fld = scenes.planted_field(svo, knot, seed=0)             # device SDF at corners
    return knot, svo, fld


def query_points(knot, n: int, seed: int = 0) -> np.ndarray:
    """2:2:1 surface / near / uniform mixture (sampling.py:159-192) over the knot."""
    from paper_2101_10994_b200 import scenes
    rng = np.random.default_rng(seed)
    n_uni = n // 5
    n_near = (2 * n) // 5
    n_surf = n - n_near - n_uni
    surf = scenes.knot_samples(knot, n_surf + n_near, seed=seed + 1)
    near = np.clip(surf[n_surf:] + 0.01 * rng.standard_normal((n_near, 3)), -1.0, 1.0)
    uni = rng.uniform(-1.0, 1.0, size=(n_uni, 3))
    return np.concatenate([surf[:n_surf], near, uni]).astype(np.float32).astype(np.float64)


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) >= 7:
                    self.rows.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ the reference package

REF_DIR = os.path.join(ROOT, "baseline", "_ref")
REF_INPUTS = os.path.join(ROOT, "bench_data", "knot_l5_ref.npz")
SAMPLE_ROW_STRIDE = 3   # cpu_baseline: every 3rd image row (240 of 720)


class Reference:
    """The unmodified reference package (`octfield`, pip-installed into
    baseline/_ref by `pip install --target baseline/_ref`), its modules by
    name. Nothing of ours is imported on this path."""

    def __init__(self):
        import importlib
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        self.pkg = importlib.import_module("octfield")
        for name in ("octree", "field", "traversal", "render", "trainer", "sampling"):
            setattr(self, name, importlib.import_module("octfield." + name))
        self.path = os.path.dirname(self.pkg.__file__)


def load_reference():
    """Reference() when baseline/_ref holds the package, else None."""
    if not os.path.isdir(os.path.join(REF_DIR, "octfield")) or not os.path.exists(REF_INPUTS):
        return None
    return Reference()


def ref_workload(ref: Reference):
    """configs[1]'s octree and planted field built by the reference itself
    from bench_data/knot_l5_ref.npz (written by the reference,
    tools/make_ref_inputs.py): build_octree over the finest voxel centres
    with corner_test=False reproduces the full build (checked there), then
    new_field(seed=0) and the Appendix A planting."""
    OT, F = ref.octree, ref.field
    z = np.load(REF_INPUTS)
    L, r0 = int(z["max_level"]), int(z["r0"])
    res = r0 << L
    codes = z["finest_codes"]
    centres = OT.cell_origin(OT.morton_decode(codes), res) + 0.5 * (2.0 / res)
    svo = OT.build_octree(None, L, centres, r0=r0, corner_test=False)
    assert [svo.voxel_count(lv) for lv in range(L + 1)] == [int(v) for v in z["voxels"]]
    fld = F.new_field(svo, seed=0)
    planted = z["planted"]
    for lv in range(1, L + 1):
        rows = np.unique(svo.levels[lv].corners)
        fld.Z[rows, lv - 1] = planted[rows]
        d = fld.decoders[lv - 1]
        d.W1[0:2, :] = 0.0
        d.b1[0:2] = 0.0
        d.W1[0, 3 + lv - 1] = 1.0
        d.W1[1, 3 + lv - 1] = -1.0
        d.W2[:] = 0.0
        d.W2[0, 0] = 1.0
        d.W2[0, 1] = -1.0
        d.b2[:] = 0.0
    return svo, fld


def ref_camera(ref: Reference, width=WIDTH, height=HEIGHT):
    R = ref.render
    return R.Camera(np.array(CAM["position"]), np.array(CAM["look_at"]), np.array(CAM["up"]), CAM["fov_y_deg"],
                    width, height)


def ref_row_sample(ref: Reference, fld, rows: np.ndarray, workers: int):
    """The reference's own render() (render.py:342-448, unmodified) over the
    rays of the given image rows: a Camera whose rays() returns those rows'
    rays (pixel-centre rays of the full 1280x720 camera), and the module seam
    `render.ray_trace_octree` wrapped to keep the final list -- the way the
    reference's tests patch its seams. Returns (seconds, rays, final list,
    report)."""
    R, T = ref.render, ref.traversal
    full = ref_camera(ref).rays()
    idx = (rows[:, None] * WIDTH + np.arange(WIDTH)[None, :]).ravel()
    bundle = T.RayBundle(full.origins[idx], full.directions[idx])

    class RowCamera(R.Camera):
        def rays(self):
            return bundle

    cam = RowCamera(np.array(CAM["position"]), np.array(CAM["look_at"]), np.array(CAM["up"]), CAM["fov_y_deg"],
                    WIDTH, len(rows))
    kept = {}
    orig = R.ray_trace_octree

    def keep(*a, **k):
        out = orig(*a, **k)
        kept["final"] = out[-1]
        return out

    R.ray_trace_octree = keep
    try:
        t0 = time.perf_counter()
        _, rep = R.render(cam, fld, R.RenderConfig(workers=workers))
        secs = time.perf_counter() - t0
    finally:
        R.ray_trace_octree = orig
    return secs, len(idx), kept["final"], rep, idx


def compare_lists(ours, theirs, idx, n_total: int) -> dict:
    """Our render path's final list (global ray ids) against the reference's
    ray_trace_octree final list over the rays idx (sample-local ids): equal
    entries, in order, t_enter / t_exit as fp64 bit patterns."""
    pos = np.full(n_total, -1, dtype=np.int64)
    pos[idx] = np.arange(len(idx))
    sel = pos[ours.rays] >= 0
    g_r, g_v = pos[ours.rays[sel]], ours.voxels[sel]
    g_a, g_b = ours.t_enter[sel], ours.t_exit[sel]
    t_r = np.asarray(theirs.rays, dtype=np.int64)
    t_v = np.asarray(theirs.voxels, dtype=np.int64)
    n = len(idx)
    gc, tc = np.bincount(g_r, minlength=n), np.bincount(t_r, minlength=n)
    bad = gc != tc
    if not bad.any():
        same = ((g_v == t_v) & (g_a.view(np.int64) == np.asarray(theirs.t_enter).view(np.int64))
                & (g_b.view(np.int64) == np.asarray(theirs.t_exit).view(np.int64)))
        bad[t_r[~same]] = True
    return {"against": "reference traversal.ray_trace_octree (unmodified)", "rays": int(n),
            "pairs": int(len(t_r)), "mismatched_rays": int(bad.sum())}


def oracle_tree(svo):
    from oracle import nglod_oracle as O
    L = svo.max_level
    return O.OracleOctree(
        r0=svo.r0, max_level=L, codes=[svo.levels[lv].codes for lv in range(L + 1)],
        parents=[svo.levels[lv].parents for lv in range(L + 1)],
        corners=[None] + [svo.levels[lv].corners for lv in range(1, L + 1)],
        corner_offsets=svo.corner_offsets, corner_count=svo.corner_count,
        region_lo=svo.region.lo, region_hi=svo.region.hi, virtual_codes=list(svo.virtual_codes))


def same_workload(ref_svo, ref_fld, svo, fld) -> bool:
    """Our workload (device build + device-planted field) equals the
    reference's, array for array."""
    for lv in range(svo.max_level + 1):
        if not np.array_equal(ref_svo.levels[lv].codes, svo.levels[lv].codes):
            return False
        if lv and not np.array_equal(ref_svo.levels[lv].corners, svo.levels[lv].corners):
            return False
    if not np.array_equal(np.asarray(ref_fld.Z, np.float32), np.asarray(fld.Z, np.float32)):
        return False
    return all(np.array_equal(a.W1, b.W1) and np.array_equal(a.b1, b.b1) and np.array_equal(a.W2, b.W2)
               and np.array_equal(a.b2, b.b2) for a, b in zip(ref_fld.decoders, fld.decoders))


# ------------------------------------------------------------------ our arm

def max_over_ranks(x: float, dev) -> float:
    """The largest per-rank value (device-timed durations: max over ranks).
    gloo (NG_DIST_BACKEND=gloo, several ranks on one GPU) reduces CPU tensors."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    if dist.get_backend() == "gloo":
        t = t.cpu()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args, rank: int, world: int):
    import torch
    import paper_2101_10994_b200 as ng
    from paper_2101_10994_b200.field import forward_levels_device
    from paper_2101_10994_b200.parallel import TiledRenderer
    from paper_2101_10994_b200.render import resolve_config, resolve_lod

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        # NG_DIST_BACKEND=gloo lets several ranks share one GPU to exercise the
        # multi-rank path on a single-GPU box; timed runs use NCCL
        backend = os.environ.get("NG_DIST_BACKEND", "nccl")
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    knot, svo, fld = build_workload()
    cam = ng.Camera(CAM["position"], CAM["look_at"], CAM["up"], CAM["fov_y_deg"], WIDTH, HEIGHT)
    config = ng.RenderConfig()
    lod = resolve_lod(cam, fld, config)
    cfg = resolve_config(fld, config, lod)
    # N = 1: one band covering the frame; N > 1: interleaved 8-row bands per
    # rank + one NCCL all-gather of the colour tiles inside the timed step.
    # Frames go `batch` per launch sequence (ng_render_batch: one traversal
    # and one march over every frame's rays, so one frame's longest rays
    # overlap the other frames' work); a step is still one frame.
    B = max(1, min(args.batch, 16))
    tiles = TiledRenderer(fld, WIDTH, HEIGHT, batch=B)
    sess = tiles.sess
    n_levels = cfg.trace_level + svo.device.n_virtual  # index of the final hit count
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def step(k):
        tiles.enqueue([cam] * k, cfg)
        if world > 1:
            return tiles.gather(("color",), dst=0, frames=k)
        return None

    # settle capacities (two-phase sizing) for a full batch before timing
    tiles.render_batch([cam] * B, config)
    img, visible_all, evals_all = tiles.render(cam, config)
    for _ in range(args.warmup):
        step(B)
    torch.cuda.synchronize()

    # the steps split evenly over the fewest launches of at most B frames
    # (20 steps at B = 16: two launches of 10, not 16 + a short tail of 4)
    n_launch = max(1, -(-args.steps // B))
    sizes = [args.steps // n_launch + (1 if i < args.steps % n_launch else 0) for i in range(n_launch)]
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) for _ in sizes]
    for e in ev:
        for x in e:
            x.record()  # materialise handles
    with ClockSampler(dev.index) as clocks:
        t_load = time.perf_counter()
        while time.perf_counter() - t_load < 1.0:  # steady load so the sampler sees clocks under load
            step(B)
            torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        for k, e in zip(sizes, ev):
            flush.zero_()  # L2 flush between launches (outside the timed events)
            e0, e_march0, e_march1, e1 = e
            sess.ws.ev_march_begin = e_march0.cuda_event
            sess.ws.ev_trace_done = e_march1.cuda_event
            e0.record()
            step(k)
            e1.record()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
    sess.ws.ev_march_begin = None
    sess.ws.ev_trace_done = None
    launch_ms = [a.elapsed_time(b) for a, _, _, b in ev]
    march_all = [a.elapsed_time(b) for _, a, b, _ in ev]
    full = [i for i, k in enumerate(sizes) if k == sizes[-1]]
    frame_ms = [launch_ms[i] / sizes[i] for i in full]
    march_ms = [march_all[i] for i in full]
    st = sess.read_stats()
    assert not st.overflow and st.counters.evals_missing_level == 0 and st.counters.nonfinite_inputs == 0
    trace_evals = int(tiles.frame["evals"][:WIDTH * len(tiles.layout[rank])].sum().item())  # frame 0 of the batch
    ms_local = sum(launch_ms) / args.steps
    if world > 1:
        ms_local = max_over_ranks(ms_local, dev)
    # one frame per launch (the latency of a frame alone), same timing
    lat = TiledRenderer(fld, WIDTH, HEIGHT)
    lat.render(cam, config)
    lat_ms = _time_tiled(lat, cam, cfg, max(3, min(args.steps, 20)), flush, world)
    # the last timed frame's per-ray voxel lists (render path), checked
    # against the reference's traversal in the cpu_baseline leg
    final = lat.sess.final_list(MAX_LEVEL) if world == 1 else None
    st = lat.sess.read_stats()  # one frame's list lengths
    del lat
    res = {
        "_final": final, "batch": B, "launches": len(sizes), "frames_per_launch": sizes,
        "ms_per_step": ms_local, "frame_ms": frame_ms, "march_ms": march_ms, "trace_evals": trace_evals,
        "frame_latency_ms": lat_ms,
        "total_evals": evals_all, "visible": visible_all, "clocks": clocks.summary(),
        "pairs": [int(st.pairs[i]) for i in range(n_levels + 1)], "active_rays": int(st.active_rays),
    }
    # presummed feature tables: built once per field and (level, output levels),
    # outside the per-frame work; their one-off cost is reported here
    dfield = fld.device
    if dfield.presum is not None:
        key = dfield._presum_key
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record()
        tables, _owner = dfield.build_presum(svo, *key)
        p1.record()
        torch.cuda.synchronize()
        res["presum"] = {"level": key[0], "out_mask": key[1], "build_ms": p0.elapsed_time(p1),
                         "table_bytes": int(tables.numel() * 4)}
        del tables, _owner

    # ---- end to end through the public API: host camera in, colour image out
    e2e_steps = max(3, min(args.steps, 20))
    if world == 1:
        # warm-up covers the frame-graph captures (render.py: a launch key is
        # captured on its second sight; consecutive frames alternate buffers)
        e2e_steps = max(3 * B, min(args.steps, 24))  # (three launches: the readback pipeline fills)
        for _ in range(6):
            fb, _r = ng.render(cam, fld, config)
            _ = fb.color
        for _ in range(2):  # (its launch graphs: a few buffer sets)
            for fb, _r in ng.render_frames([cam] * e2e_steps, fld, config, batch=B):
                _ = fb.color
        torch.cuda.synchronize()
        # render_frames: `batch` frames per launch sequence; each launch's
        # colour images and statistics come back while the next one runs
        # (double-buffered readback); every frame's image is still copied to
        # the host inside the timed region
        batches = []
        for _ in range(3):  # the median of three runs (host jitter)
            t0 = time.perf_counter()
            for fb, rep in ng.render_frames([cam] * e2e_steps, fld, config, batch=B):
                img = fb.color
            batches.append((time.perf_counter() - t0) / e2e_steps)
        e2e_s = statistics.median(batches)
        assert rep.visible % visible_all == 0  # (a batch's report: its frames' total)
        d2h = int(img.nbytes)
    else:
        for _ in range(2):
            img_d = tiles.render_batch([cam] * B, config, dst=0)[0]
            if img_d is not None:
                img_d.cpu()
        torch.distributed.barrier()
        launches = max(2, (min(args.steps, 24) + B - 1) // B)
        # rank 0 copies the gathered images into pinned host memory (a
        # pageable .cpu() of B frames ran at a few GB/s)
        pin = torch.empty((B, HEIGHT, WIDTH, 3), dtype=torch.uint8, pin_memory=True) if rank == 0 else None
        t0 = time.perf_counter()
        img = np.zeros((B, HEIGHT, WIDTH, 3), np.uint8)
        for _ in range(launches):
            img_d, _v, _e = tiles.render_batch([cam] * B, config, dst=0)
            if img_d is not None:
                pin.copy_(img_d, non_blocking=True)
                torch.cuda.current_stream().synchronize()
                img = pin.numpy()
        e2e_s = (time.perf_counter() - t0) / (launches * B)
        e2e_s = max_over_ranks(e2e_s, dev)
        d2h = int(img.nbytes) // B
    res["e2e"] = {"value": 1.0 / e2e_s, "unit": "frames/s",
                  "h2d_bytes_per_step": _sizeof("NgCamera") + _sizeof("NgRenderCfg"),
                  "d2h_bytes_per_step": d2h + _sizeof("NgFrameStats"),
                  "api": f"render_frames(batch={B}) (a launch's readback overlaps the next launch)" if world == 1
                  else f"TiledRenderer.render_batch ({B} frames), colour gathered to rank 0 and copied to pinned host "
                       "memory"}

    # ---- batched SDF query (configs[2]): forward L = 1..5 over 2^24 points,
    # sharded by point range across ranks (no exchange)
    if not args.no_query:
        res["query"], res["_query_pts"] = query_leg(knot, svo, fld, dev, flush, rank, world)
    # ---- configs[3] / configs[4] at 1920x1080 (tiled across the ranks when N > 1)
    if not args.no_extra:
        res["extra"] = extra_configs(args, world, dev, knot)

    # ---- training step: one epoch of loss + backward + Adam,
    # batch 512, fp64 masters, random-init LOD5 field (rank 0 / N = 1 only: the
    # reference trains in one process)
    if not args.no_train and world == 1:
        res["train"] = train_leg(knot, svo, dev, flush)
    res["_svo"], res["_fld"] = svo, fld
    return res


QUERY_LEVELS = [1, 2, 3, 4, 5]
QUERY_BYTES_BASE = 32   # SURVEY.md 8d, configs[2]: 32 + 1,064 k B per point (k present levels)
QUERY_TIMED = 9


def query_leg(knot, svo, fld, dev, flush, rank: int, world: int):
    """configs[2]: forward L = 1..5 over 2^24 points (2:2:1 mix), through
    the device entry (points resident in HBM) and end to end through the
    public NeuralField.forward_levels (numpy in, numpy out). Median and
    spread of the timed calls; the roofline counts the present levels k of
    every point with the query's own device counters."""
    import torch
    from paper_2101_10994_b200.field import EvalCounter, forward_levels_device
    pts_h = query_points(knot, QUERY_POINTS)
    share = QUERY_POINTS // world
    mine = np.ascontiguousarray(pts_h[rank * share:(rank + 1) * share])
    pts = torch.from_numpy(mine).to(dev)
    # sum of k: decoded (point, L) rows minus rows whose level-L voxel is
    # missing (EvalCounter semantics, field.py:79-90, 194-218)
    cnt = EvalCounter()
    out = forward_levels_device(svo, fld.device, pts, QUERY_LEVELS, counter=cnt)
    sum_k = cnt.decoder_evals - cnt.evals_missing_level
    torch.cuda.synchronize()
    qe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(QUERY_TIMED)]
    # the output stays resident (out=): a fresh 671 MB allocation per call
    # while the previous result is alive made single calls take up to 4x
    # longer (profiles/r02/query_kernel_probe.log)
    for a, b in qe:
        flush.zero_()
        a.record()
        forward_levels_device(svo, fld.device, pts, QUERY_LEVELS, out=out)
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in qe)
    q_ms = statistics.median(ms)
    if world > 1:
        q_ms = max_over_ranks(q_ms, dev)
    del out
    algo = share * QUERY_BYTES_BASE + EVAL_BYTES_PER_LEVEL * sum_k
    achieved = algo / (ms[len(ms) // 2] * 1e-3) / 1e9
    peak = _peak_hbm()
    line = {"metric": "Mpoints/sec batched SDF query (forward L=1..5, 2^24 points, 2:2:1 mix)",
            "value": share * world / q_ms / 1e3, "unit": "Mpoints/s", "ms_median": q_ms,
            "ms_min": ms[0], "ms_max": ms[-1], "timed_calls": len(ms),
            "mean_levels_k": sum_k / share,
            "roofline": {"bound": "hbm", "kernel": "k_query_tc (+ the decoder-staging k_query_tiles, one call)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": _traffic("query_traffic.json"), "algorithmic_bytes": algo,
                         "note": f"{QUERY_BYTES_BASE} + {EVAL_BYTES_PER_LEVEL} k B per point (SURVEY.md 8d), "
                                 "k counted on the device; the call's median event time; peak = measured hbm_gbs. "
                                 "The rows are served from L2 (traffic = the call's DRAM bytes), so frac can pass 1; "
                                 "the binding roof is the L2 random-row gather peak (l2_frac)"}}
    l2 = _l2_peak()
    if l2:
        line["roofline"]["l2_gather_peak"] = l2
        line["roofline"]["l2_frac"] = achieved / l2
    # end to end: the public API with host arrays (pageable numpy in, numpy out)
    e2e = []
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        host_out = fld.forward_levels(mine, QUERY_LEVELS)
        if i:
            e2e.append(time.perf_counter() - t0)
    e2e_s = statistics.median(e2e)
    if world > 1:
        e2e_s = max_over_ranks(e2e_s, dev)
    line["e2e"] = {"value": share * world / e2e_s / 1e6, "unit": "Mpoints/s",
                   "h2d_bytes_per_step": int(mine.nbytes), "d2h_bytes_per_step": int(host_out.nbytes),
                   "note": "NeuralField.forward_levels(numpy points) -> numpy (n, 5) fp64, median of 3"}
    return line, pts_h


TRAIN_POINTS = 500_000   # TrainConfig.points_per_epoch default (trainer.py:39)
TRAIN_BATCH = 512        # TrainConfig.batch_size default (trainer.py:40)


def train_leg(knot, svo, dev, flush):
    import torch
    import paper_2101_10994_b200 as ng
    from paper_2101_10994_b200.trainer import DeviceTrainer
    fld = ng.new_field(svo, seed=0)
    pts_h = query_points(knot, TRAIN_POINTS, seed=1)
    pts = torch.from_numpy(pts_h).to(dev)
    dist = knot.device_eval(pts)
    dist_h = dist.cpu().numpy()
    work = ng.NeuralField(svo, fld.Z.astype(np.float64), [d.astype(np.float64) for d in fld.decoders])
    tr = DeviceTrainer(work, TRAIN_BATCH)
    act = list(range(1, MAX_LEVEL + 1))
    tr.run_epoch(pts, dist, act, True, 1e-3)  # warm-up epoch (977 Adam steps)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
    for a, b in ev:
        flush.zero_()
        a.record()
        tr.run_epoch(pts, dist, act, True, 1e-3)
        b.record()
    torch.cuda.synchronize()
    ms = min(a.elapsed_time(b) for a, b in ev)
    assert tr.diverged_at() < 0
    # end to end: host points in (pinned), per-level epoch losses out
    pin_p = torch.from_numpy(pts_h).pin_memory()
    pin_d = torch.from_numpy(dist_h).pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2):
        dp = pin_p.to(dev, non_blocking=True)
        dd = pin_d.to(dev, non_blocking=True)
        tr.run_epoch(dp, dd, act, True, 1e-3)
        losses = tr.level_sums.cpu().numpy() / TRAIN_POINTS
    e2e_s = (time.perf_counter() - t0) / 2
    # the public API: ng.train for one epoch, including the epoch sampler
    # (numpy random streams on the host, surface tracing + distances on the GPU)
    t0 = time.perf_counter()
    _, hist = ng.train(knot, fld, ng.TrainConfig(epochs=1, points_per_epoch=TRAIN_POINTS, batch_size=TRAIN_BATCH))
    api_s = time.perf_counter() - t0
    n_batches = (TRAIN_POINTS + TRAIN_BATCH - 1) // TRAIN_BATCH
    return {"metric": "Mpoints/sec training step (loss + backward + Adam, fp64 masters)",
            "value": TRAIN_POINTS / ms / 1e3, "unit": "Mpoints/s", "ms_per_epoch": ms,
            "us_per_batch": ms * 1e3 / n_batches, "points_per_epoch": TRAIN_POINTS, "batch_size": TRAIN_BATCH,
            "adam_steps_per_epoch": n_batches, "dtype": "fp64",
            "workload": "LOD5 torus-knot octree, new_field(seed=0) m=32 h=128, 2:2:1 knot mix, joint schedule",
            "launches_per_batch": 7, "level_losses": [float(x) for x in losses],
            "e2e": {"value": TRAIN_POINTS / e2e_s / 1e6, "unit": "Mpoints/s",
                    "h2d_bytes_per_step": int(pts_h.nbytes + dist_h.nbytes), "d2h_bytes_per_step": 8 * MAX_LEVEL},
            "api_epoch": {"value": TRAIN_POINTS / api_s / 1e6, "unit": "Mpoints/s", "seconds": api_s,
                          "note": "ng.train(knot, field, TrainConfig(epochs=1)) wall clock, incl. the epoch sampler"},
            "_pts": pts_h, "_dist": dist_h, "_fld": work}


def _time_tiled(tiles, cam, cfg, steps, flush, world):
    """Median ms per frame over `steps` launches of `tiles.batch` frames of
    `cam` each (L2 flushed before each launch; N > 1: with the gather)."""
    import torch
    k = tiles.batch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for _ in range(2):
        tiles.enqueue([cam] * k, cfg)
    torch.cuda.synchronize()
    for a, b in ev:
        flush.zero_()
        a.record()
        tiles.enqueue([cam] * k, cfg)
        if world > 1:
            tiles.gather(("color",), dst=0, frames=k)
        b.record()
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in ev) / k
    if world > 1:
        ms = max_over_ranks(ms, flush.device)
    return ms


def extra_configs(args, world, dev, knot):
    """configs[3]: LOD6 1920x1080 (image bands + NCCL gather when N > 1);
    configs[4]: continuous LOD 4.5 with shadow rays at 1920x1080."""
    import torch
    import paper_2101_10994_b200 as ng
    from paper_2101_10994_b200 import scenes
    from paper_2101_10994_b200.parallel import TiledRenderer
    from paper_2101_10994_b200.render import resolve_config, resolve_lod
    _, samples = knot_scene()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    out = {}
    svo6 = ng.build_octree(knot, 6, samples)
    fld6 = scenes.planted_field(svo6, knot, seed=0)
    cam = ng.Camera(CAM["position"], CAM["look_at"], CAM["up"], CAM["fov_y_deg"], 1920, 1080)
    steps = max(3, min(args.steps, 10))
    for name, fld, config in (
            ("configs[3] LOD6 1920x1080", fld6, ng.RenderConfig()),
            ("configs[4] LOD4.5 + shadow rays 1920x1080", fld6, ng.RenderConfig(lod=4.5, shadows=True))):
        cfg = resolve_config(fld, config, resolve_lod(cam, fld, config))
        tiles = TiledRenderer(fld, 1920, 1080)
        img, visible, evals = tiles.render(cam, config)
        st = tiles.sess.read_stats()
        lat = _time_tiled(tiles, cam, cfg, steps, flush, world)
        del tiles
        B = max(1, min(args.batch, 16))
        tiles = TiledRenderer(fld, 1920, 1080, batch=B)
        tiles.render_batch([cam] * B, config)  # capacities for the batch
        ms = _time_tiled(tiles, cam, cfg, max(3, steps // 2), flush, world)
        del tiles
        out[name] = {"frames_per_sec": 1000.0 / ms, "ms_per_frame": ms, "frames_per_launch": B,
                     "frame_latency_ms": lat, "visible": visible, "decoder_evals": evals,
                     "shadowed_local": int(st.shadowed), "voxels_finest": svo6.voxel_count(6), "n_gpus": world}
    return out


def _ref(x):
    import ctypes
    return ctypes.byref(x)


def _sizeof(name):
    import ctypes
    from paper_2101_10994_b200 import _lib
    return ctypes.sizeof(getattr(_lib, name))


DTYPE = ("fp64 traversal, march control and shading; fp32 feature tables; decoder layer 1 as a bf16x3 split "
         "on tcgen05 with fp32 accumulation, layer 2 fp32")
DATA = "synthetic: (2,3) torus-knot polyline SDF, planted field (SURVEY.md Appendix A), random-init remainder"
VOXELS = [30, 134, 450, 2150, 11946, 72125]   # knot LOD5 per level (the reference's build)


def line_config(world: int) -> dict:
    """The `config` of both arms' lines (identical for the same N)."""
    return {"workload": "configs[1]: LOD5 torus-knot octree, 1280x720 sparse sphere trace + normals + Lambert shading",
            "resolution": [WIDTH, HEIGHT], "lod": MAX_LEVEL, "voxels": VOXELS, "camera": CAM,
            "parallelism": f"tiles{world}" + (" (8-row bands, NCCL all-gather of the colour tiles)" if world > 1
                                              else ""),
            "frames": "a sequence of frames of this camera (a static view); one step = one frame",
            "l2": "flushed between GPU launch sequences (256 MiB write)"}


def spawn_ranks(args) -> int:
    """--gpus N > 1 without a torchrun environment: run N ranks of this
    script under torch.distributed.run on this node and pass their exit
    code on (rank 0 prints the line)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.impl == "reference":
        return run_reference(args, rank, world)
    res = run_ours(args, rank, world)
    if rank != 0:
        return
    ms = res["ms_per_step"]
    fps = 1000.0 / ms  # one full 1280x720 frame per step, split across the ranks
    march = statistics.median(res["march_ms"])
    # with the presummed tables (csrc/presum.cu) an evaluation reads one
    # level's node, corner ids and 8 table rows per output level; without
    # them, every level 1..L
    levels_read = 1 if res.get("presum") else MAX_LEVEL
    bytes_per_eval = EVAL_BYTES_BASE + EVAL_BYTES_PER_LEVEL * levels_read
    # the march launch also evaluates the normal probes (NG_FUSED_PROBES, default)
    fused = os.environ.get("NG_FUSED_PROBES", "1") != "0"
    # a full launch marches `batch` frames of the same camera
    march_evals = (res["total_evals"] if fused else res["trace_evals"]) * res["frames_per_launch"][-1]
    algo_bytes = march_evals * bytes_per_eval
    peak = _peak_hbm()
    achieved = algo_bytes / (march * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": DTYPE, "data": DATA, "config": line_config(world),
        "mrays_per_sec": WIDTH * HEIGHT * fps / 1e6,
        "frame": {"visible": res["visible"], "trace_evals": res["trace_evals"],
                  "total_evals": res["total_evals"], "pairs_per_level": res["pairs"],
                  "active_rays": res["active_rays"], "march_ms_median": march,
                  "frame_ms_median": statistics.median(res["frame_ms"]), "voxels": _voxel_counts(res["_svo"]),
                  "frames_per_launch": res["frames_per_launch"], "launch_march_ms_median": march},
        "frame_latency_ms": res["frame_latency_ms"],
        "frame_latency_note": "one frame per launch sequence (TiledRenderer without batching), same timing: "
                              "what a single frame takes alone",
        "e2e": res["e2e"],
        "gpu_launches": res["launches"] * (_launches_per_frame(res["_svo"]) + (world + 2 if world > 1 else 0)),
        "roofline": {"bound": "hbm", "kernel": "k_march (sphere-trace march + normal probes, fused gather + MLP)"
                     if fused else "k_march (sphere-trace march, fused gather + MLP)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": _march_traffic(res["frames_per_launch"][-1]),
                     "algorithmic_bytes": algo_bytes,
                     "evals": march_evals,
                     "note": f"{bytes_per_eval} B per eval x the launch's evals ({levels_read} level(s) read per eval: "
                             "presummed S_L rows (SURVEY.md 8d per-level bytes)); peak = measured hbm_gbs"},
        "clocks": res["clocks"],
        "presum": res.get("presum"),
    }
    l2 = _l2_peak()
    if l2:
        line["roofline"]["l2_gather_peak"] = l2
        line["roofline"]["l2_frac"] = achieved / l2
    if "query" in res:
        line["query"] = res["query"]
    if "extra" in res:
        line["configs_3_4"] = res["extra"]
    if "train" in res:
        line["train"] = {k: v for k, v in res["train"].items() if not k.startswith("_")}
    if not args.no_cpu and world == 1:
        cpu, check = cpu_baseline(res)
        line["cpu_baseline"] = cpu
        if check is not None:
            line["traversal_check"] = check
    print(json.dumps(line))


def _voxel_counts(svo):
    return [svo.voxel_count(lv) for lv in range(svo.max_level + 1)]


def _launches_per_frame(svo):
    # zeroing, the tile traversal (all levels, frame defaults, work list),
    # the march (normals as probe items inside it, statistics); the
    # level-by-level traversal (NG_TILE_TRAVERSE=0) adds the camera-ray
    # kernel, one pass per level and the histogram + scatter,
    # NG_FUSED_PROBES=0 the normals pass (cf. profiles/r01_tiles/launch_shares.md)
    levels = os.environ.get("NG_TILE_TRAVERSE", "1") == "0"
    fused = os.environ.get("NG_FUSED_PROBES", "1") != "0"
    n = 1 + 1 + 1  # (the march's last CTA writes the frame statistics)
    if levels:
        n += 1 + (MAX_LEVEL + svo.device.n_virtual) - 1 + 2
    if not fused:
        n += 2  # normals pass, statistics kernel
    return n


def _peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0  # fallback figure (B200_PROFILING.md)


def _l2_peak():
    """Random 128-byte row gather bandwidth out of L2 (GB/s), measured by
    tools/micro/l2_gather.cu and committed under profiles/."""
    try:
        with open(os.path.join(ROOT, "profiles", "l2_gather_peak.json")) as fh:
            return float(json.load(fh)["gbs"])
    except Exception:
        return None


def _march_traffic(frames: int):
    """k_march DRAM bytes per launch of `frames` frames: the committed ncu
    capture's bytes per frame times the frames (the capture may have been
    of a different batch size)."""
    p = os.path.join(ROOT, "profiles", "march_traffic.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d["dram_bytes_per_launch"] / d.get("frames_per_launch", 1) * frames
    except Exception:
        return None


def _traffic(name="march_traffic.json"):
    """dram bytes per launch from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", name)
    try:
        with open(p) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    except Exception:
        return None


def cpu_baseline(res):
    """The reference itself (baseline/_ref, unmodified) on the host cores:
    its render() over every 3rd image row of the same frame (~1/3 of the
    work), forward L = 1..5 over 65,536 of the query points and 6 training
    batches, each scaled to the line's unit. The same row sample checks our
    render path's per-ray voxel lists against the reference's
    ray_trace_octree bit for bit, and the oracle counts the sample's
    near-tie slab decisions. Returns (cpu_baseline, traversal_check)."""
    ref = load_reference()
    if ref is None:
        return {"unavailable": "reference not installed in baseline/_ref (or bench_data missing)"}, None
    workers = os.cpu_count() or 1
    ref_svo, ref_fld = ref_workload(ref)
    identical = same_workload(ref_svo, ref_fld, res["_svo"], res["_fld"])
    rows = np.arange(SAMPLE_ROW_STRIDE // 2, HEIGHT, SAMPLE_ROW_STRIDE)
    secs, n, ref_final, rep, idx = ref_row_sample(ref, ref_fld, rows, workers)
    fps = (n / (WIDTH * HEIGHT)) / secs
    out = {"value": fps, "unit": "frames/s", "cores": workers, "kind": "reference",
           "sample": f"reference render() over every {SAMPLE_ROW_STRIDE}rd row ({n} rays) of the 1280x720 frame, "
                     f"{secs:.1f} s, scaled to frames/s",
           "reference": ref.path, "workload_identical": identical}
    check = None
    if res.get("_final") is not None:
        check = compare_lists(res["_final"], ref_final, idx, WIDTH * HEIGHT)
        from oracle import nglod_oracle as O
        o, d = O.camera_rays(CAM["position"], CAM["look_at"], CAM["up"], CAM["fov_y_deg"], WIDTH, HEIGHT)
        ties = []
        O.traverse(oracle_tree(res["_svo"]), o[idx], d[idx], MAX_LEVEL, ties=ties)
        check["near_tie_decisions"] = int(sum(a for a, _ in ties))
        check["decisions"] = int(sum(b for _, b in ties))
        check["near_tie_rel"] = O.TIE_REL
        check["sample"] = f"every {SAMPLE_ROW_STRIDE}rd row of the last timed frame"
    if "_query_pts" in res:
        pts = res["_query_pts"][:: max(1, QUERY_POINTS // 65536)][:65536]
        qs = ref_query_sample(ref, ref_fld, pts, workers)
        out["query"] = {"value": len(pts) / qs / 1e6, "unit": "Mpoints/s", "cores": workers,
                        "sample": f"reference forward(x, L) for L = 1..5 over {len(pts)} points in 8,192-point chunks "
                                  f"on {workers} threads, {qs:.1f} s"}
    if "train" in res:
        secs_t, npts = ref_train_sample(ref, ref_fld, res["train"])
        out["train"] = {"value": npts / secs_t / 1e6, "unit": "Mpoints/s", "cores": 1,
                        "sample": f"{npts // TRAIN_BATCH} reference Adam steps of batch {TRAIN_BATCH} "
                                  f"(trainer._batch_pass + adam_step, fp64), {secs_t:.1f} s"}
    return out, check


def ref_query_sample(ref: Reference, fld, pts: np.ndarray, workers: int) -> float:
    """the reference's training-forward path, forward(x, L)
    for L = 1..5, over chunks on a thread pool (trainer.py:254-279 style)."""
    from concurrent.futures import ThreadPoolExecutor
    F = ref.field
    chunks = [pts[s:s + 8192] for s in range(0, len(pts), 8192)]

    def run(c):
        return [F.forward(fld.svo, fld.Z, fld.decoders, c, L)[0] for L in QUERY_LEVELS]

    t0 = time.perf_counter()
    with ThreadPoolExecutor(workers) as pool:
        list(pool.map(run, chunks))
    return time.perf_counter() - t0


def ref_train_sample(ref: Reference, fld, tr, batches: int = 6):
    """The reference's inner training loop (trainer.py:210-229:
    _batch_pass, adam_step) on the bench's random-init field and points,
    single-threaded, a few batches."""
    T = ref.trainer
    F = ref.field
    src = tr["_fld"]
    work = F.NeuralField(fld.svo, np.array(src.Z, dtype=np.float64),
                         [F.Decoder(d.W1.astype(np.float64), d.b1.astype(np.float64), d.W2.astype(np.float64),
                                    d.b2.astype(np.float64)) for d in src.decoders])
    params = {"Z": work.Z}
    for i, d in enumerate(work.decoders):
        for nm in ("W1", "b1", "W2", "b2"):
            params[f"decoder{i + 1}.{nm}"] = getattr(d, nm)
    state = T.AdamState.for_params(params)
    act = list(range(1, MAX_LEVEL + 1))
    tags = np.zeros(TRAIN_BATCH, dtype=np.int8)
    t0 = time.perf_counter()
    for b in range(batches):
        sl = slice(b * TRAIN_BATCH, (b + 1) * TRAIN_BATCH)
        batch = ref.sampling.SampleSet(tr["_pts"][sl], tr["_dist"][sl], tags)
        _, grads, _ = T._batch_pass(work, batch, act, None)
        T.adam_step(params, T._grads_dict(grads, True), state, 1e-3)
    return time.perf_counter() - t0, batches * TRAIN_BATCH


# ------------------------------------------------------------------ reference arm

REF_TIME_BUDGET_S = 1500.0   # the driver's limit for this step is 1,800 s


def run_reference(args, rank: int, world: int):
    """The unmodified reference (`octfield` from baseline/_ref) through its
    public render() on the host cores (RenderConfig(workers=os.cpu_count())),
    one WHOLE 1280x720 frame per step, on the configs[1] octree and planted
    field the reference built itself (bench_data/knot_l5_ref.npz). Rank 0
    only; nothing of ours is imported. A CPU path has nothing to warm beyond
    its first frame, so one warm-up frame is run whatever W says (both
    numbers are in the line); if the frames run slower than the driver's
    step allows, the timed frames stop early and `steps` says how many ran."""
    if rank != 0:
        return
    ref = load_reference()
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": "octfield not installed in baseline/_ref "
                                                              "(pip install --target baseline/_ref) or "
                                                              "bench_data/knot_l5_ref.npz missing"}))
        return
    workers = os.cpu_count() or 1
    t_start = time.perf_counter()
    svo, fld = ref_workload(ref)
    cam = ref_camera(ref)
    config = ref.render.RenderConfig(workers=workers)
    warm = min(args.warmup, 1)
    for _ in range(warm):
        _, rep = ref.render.render(cam, fld, config)
    times = []
    for k in range(args.steps):
        t0 = time.perf_counter()
        _, rep = ref.render.render(cam, fld, config)
        times.append(time.perf_counter() - t0)
        spent = time.perf_counter() - t_start
        if spent + statistics.mean(times) > REF_TIME_BUDGET_S:
            break
    ms = statistics.mean(times) * 1e3
    fps = 1000.0 / ms
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": len(times), "warmup": warm, "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "fp64 (the reference computes in fp64 with fp32 parameters)", "data": DATA,
        "config": line_config(world),
        "frame": {"visible": int(rep.visible), "total_evals": int(rep.evals), "ms_trace": rep.ms_trace,
                  "ms_normals": rep.ms_normals, "frame_s": times},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": workers, "kind": "reference",
                         "sample": f"whole frames: octfield.render.render() x {len(times)} (mean)",
                         "reference": ref.path},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
