"""Benchmark: frames/sec of the 1280x720 LOD5 sparse sphere trace (BASELINE.json
configs[1]) on B200, plus the batched SDF query (configs[2]) in Mpoints/sec.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0. A step is one full frame of the hot path --
camera rays, BFS traversal, persistent sphere-trace march, normals and
shading -- over the torus-knot LOD5 octree with the planted field (SURVEY.md
Appendix A; synthetic, no training). `value` is device time (CUDA events,
L2 flushed between frames); `e2e` times the public `render()` call with the
colour image read back to the host. `--impl reference` times the CPU oracle
port (the reference is pure Python; its algorithm restated in oracle/) on
bounded samples of the same workload.
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


# ------------------------------------------------------------------ CPU oracle legs

def oracle_tree(svo):
    from oracle import nglod_oracle as O
    L = svo.max_level
    return O.OracleOctree(
        r0=svo.r0, max_level=L, codes=[svo.levels[lv].codes for lv in range(L + 1)],
        parents=[svo.levels[lv].parents for lv in range(L + 1)],
        corners=[None] + [svo.levels[lv].corners for lv in range(1, L + 1)],
        corner_offsets=svo.corner_offsets, corner_count=svo.corner_count,
        region_lo=svo.region.lo, region_hi=svo.region.hi, virtual_codes=list(svo.virtual_codes))


def cpu_frame_sample(tree, fld, row_stride: int, row_offset: int = 0, workers: int | None = None):
    """Oracle render of every `row_stride`-th image row; returns (seconds, rays)."""
    from oracle import nglod_oracle as O
    workers = workers or os.cpu_count() or 1
    decs = [O.OracleDecoder(d.W1, d.b1, d.W2, d.b2) for d in fld.decoders]
    rows = np.arange(row_offset, HEIGHT, row_stride)
    idx = (rows[:, None] * WIDTH + np.arange(WIDTH)[None, :]).ravel()
    cam = dict(CAM, width=WIDTH, height=HEIGHT)
    t0 = time.perf_counter()
    O.render(tree, fld.Z, decs, cam, O.RenderParams(), ray_slice=idx, workers=workers)
    return time.perf_counter() - t0, len(idx)


def cpu_query_sample(tree, fld, pts: np.ndarray, workers: int | None = None):
    from concurrent.futures import ThreadPoolExecutor
    from oracle import nglod_oracle as O
    workers = workers or os.cpu_count() or 1
    decs = [O.OracleDecoder(d.W1, d.b1, d.W2, d.b2) for d in fld.decoders]
    chunks = [pts[s:s + 8192] for s in range(0, len(pts), 8192)]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(workers) as pool:
        list(pool.map(lambda c: O.forward_levels(tree, fld.Z, decs, c, [1, 2, 3, 4, 5]), chunks))
    return time.perf_counter() - t0


# ------------------------------------------------------------------ our arm

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
    # rank + one NCCL all-gather of the colour tiles inside the timed step
    tiles = TiledRenderer(fld, WIDTH, HEIGHT)
    sess = tiles.sess
    n_levels = cfg.trace_level + svo.device.n_virtual  # index of the final hit count
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def step():
        tiles.enqueue(cam, cfg)
        if world > 1:
            return tiles.gather_color()
        return None

    # settle capacities (two-phase sizing) before timing
    img, visible_all, evals_all = tiles.render(cam, config)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) for _ in range(args.steps)]
    for e in ev:
        for x in e:
            x.record()  # materialise handles
    with ClockSampler(dev.index) as clocks:
        t_load = time.perf_counter()
        while time.perf_counter() - t_load < 1.0:  # steady load so the sampler sees clocks under load
            step()
            torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.zero_()  # L2 flush between frames (outside the timed events)
            e0, e_march0, e_march1, e1 = ev[k]
            sess.ws.ev_march_begin = e_march0.cuda_event
            sess.ws.ev_trace_done = e_march1.cuda_event
            e0.record()
            step()
            e1.record()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
    sess.ws.ev_march_begin = None
    sess.ws.ev_trace_done = None
    frame_ms = [a.elapsed_time(b) for a, _, _, b in ev]
    march_ms = [a.elapsed_time(b) for _, a, b, _ in ev]
    st = sess.read_stats()
    assert not st.overflow and st.counters.evals_missing_level == 0 and st.counters.nonfinite_inputs == 0
    trace_evals = int(tiles.frame["evals"].sum().item())
    ms_local = sum(frame_ms) / len(frame_ms)
    if world > 1:
        t = torch.tensor([ms_local], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_local = float(t.item())
    res = {
        "ms_per_step": ms_local, "frame_ms": frame_ms, "march_ms": march_ms, "trace_evals": trace_evals,
        "total_evals": evals_all, "visible": visible_all, "clocks": clocks.summary(),
        "pairs": [int(st.pairs[i]) for i in range(n_levels + 1)], "active_rays": int(st.active_rays),
    }
    # presummed feature tables: built once per field and (level, output levels),
    # outside the per-frame work; their one-off cost is reported here
    dfield = fld.device
    if dfield.presum is not None:
        key = dfield._presum_key
        dfield._presum_key = None
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record()
        dfield.ensure_presum(svo, *key)
        p1.record()
        torch.cuda.synchronize()
        res["presum"] = {"level": key[0], "out_mask": key[1], "build_ms": p0.elapsed_time(p1),
                         "table_bytes": int(dfield.presum.numel() * 4)}

    # ---- end to end through the public API: host camera in, colour image out
    e2e_steps = max(3, min(args.steps, 20))
    if world == 1:
        # warm-up covers the frame-graph captures (render.py: a launch key is
        # captured on its second sight; consecutive frames alternate buffers)
        for _ in range(6):
            fb, _r = ng.render(cam, fld, config)
            _ = fb.color
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            fb, rep = ng.render(cam, fld, config)
            img = fb.color
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        assert rep.visible == visible_all
        d2h = int(img.nbytes)
    else:
        for _ in range(2):
            tiles.render(cam, config)[0].cpu()
        torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            img_d, _v, _e = tiles.render(cam, config)
            img = img_d.cpu()
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        t = torch.tensor([e2e_s], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
        d2h = int(img.numel())
    res["e2e"] = {"value": 1.0 / e2e_s, "unit": "frames/s",
                  "h2d_bytes_per_step": _sizeof("NgCamera") + _sizeof("NgRenderCfg"),
                  "d2h_bytes_per_step": d2h + _sizeof("NgFrameStats")}

    # ---- batched SDF query (configs[2]): forward L = 1..5 over 2^24 points,
    # sharded by point range across ranks (no exchange)
    if not args.no_query:
        pts_h = query_points(knot, QUERY_POINTS)
        share = QUERY_POINTS // world
        pts = torch.from_numpy(pts_h[rank * share:(rank + 1) * share]).to(dev)
        for _ in range(2):
            out = forward_levels_device(svo, fld.device, pts, [1, 2, 3, 4, 5])
        torch.cuda.synchronize()
        qe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(7)]
        for a, b in qe:
            flush.zero_()
            a.record()
            out = forward_levels_device(svo, fld.device, pts, [1, 2, 3, 4, 5])
            b.record()
        torch.cuda.synchronize()
        q_ms = min(a.elapsed_time(b) for a, b in qe)
        if world > 1:
            t = torch.tensor([q_ms], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            q_ms = float(t.item())
        res["query"] = {"metric": "Mpoints/sec batched SDF query (forward L=1..5, 2^24 points, 2:2:1 mix)",
                        "value": share * world / q_ms / 1e3, "unit": "Mpoints/s", "ms": q_ms}
        res["_query_pts"] = pts_h
        del out
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
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for _ in range(2):
        tiles.enqueue(cam, cfg)
    torch.cuda.synchronize()
    for a, b in ev:
        flush.zero_()
        a.record()
        tiles.enqueue(cam, cfg)
        if world > 1:
            tiles.gather_color()
        b.record()
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        t = torch.tensor([ms], device=flush.device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
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
        tiles = TiledRenderer(fld, 1920, 1080)
        img, visible, evals = tiles.render(cam, config)
        cfg = resolve_config(fld, config, resolve_lod(cam, fld, config))
        ms = _time_tiled(tiles, cam, cfg, steps, flush, world)
        st = tiles.sess.read_stats()
        out[name] = {"frames_per_sec": 1000.0 / ms, "ms_per_frame": ms, "visible": visible, "decoder_evals": evals,
                     "shadowed_local": int(st.shadowed), "voxels_finest": svo6.voxel_count(6), "n_gpus": world}
    return out


def _ref(x):
    import ctypes
    return ctypes.byref(x)


def _sizeof(name):
    import ctypes
    from paper_2101_10994_b200 import _lib
    return ctypes.sizeof(getattr(_lib, name))


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
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
    march_evals = res["total_evals"] if fused else res["trace_evals"]
    algo_bytes = march_evals * bytes_per_eval
    peak = _peak_hbm()
    achieved = algo_bytes / (march * 1e-3) / 1e9
    traffic = _traffic()
    line = {
        "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "fp32 (features, MLP) + fp64 (traversal, march control)",
        "data": "synthetic: (2,3) torus-knot polyline SDF, planted field, random-init remainder",
        "config": {"workload": "configs[1]: LOD5 torus-knot octree, 1280x720 sparse sphere trace + normals + "
                               "Lambert shading" + (f", 8-row bands over {world} B200 + NCCL all-gather"
                                                    if world > 1 else ", 1 B200"),
                   "resolution": [WIDTH, HEIGHT], "lod": MAX_LEVEL, "parallelism": f"tiles{world}",
                   "voxels": [svo_count for svo_count in _voxel_counts(res["_svo"])],
                   "l2": "flushed between frames (256 MiB write)", "camera": CAM},
        "mrays_per_sec": WIDTH * HEIGHT * fps / 1e6,
        "frame": {"visible": res["visible"], "trace_evals": res["trace_evals"],
                  "total_evals": res["total_evals"], "pairs_per_level": res["pairs"],
                  "active_rays": res["active_rays"], "march_ms_median": march,
                  "frame_ms_median": statistics.median(res["frame_ms"])},
        "e2e": res["e2e"],
        "gpu_launches": args.steps * (_launches_per_frame(res["_svo"]) + (world + 1 if world > 1 else 0)),
        "roofline": {"bound": "hbm", "kernel": "k_march (sphere-trace march + normal probes, fused gather + MLP)"
                     if fused else "k_march (sphere-trace march, fused gather + MLP)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "algorithmic_bytes": algo_bytes,
                     "evals": march_evals,
                     "note": f"{bytes_per_eval} B per eval x the launch's evals ({levels_read} level(s) read per eval: "
                             "presummed S_L rows (SURVEY.md 8d per-level bytes)); peak = measured hbm_gbs"},
        "clocks": res["clocks"],
        "presum": res.get("presum"),
    }
    if "query" in res:
        line["query"] = res["query"]
    if "extra" in res:
        line["configs_3_4"] = res["extra"]
    if "train" in res:
        line["train"] = {k: v for k, v in res["train"].items() if not k.startswith("_")}
    if not args.no_cpu and world == 1:
        line["cpu_baseline"] = cpu_baseline(res)
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


def _traffic():
    """dram bytes per k_march launch from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "march_traffic.json")
    try:
        with open(p) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    except Exception:
        return None


def cpu_baseline(res):
    """Oracle port on the host cores: every 3rd image row of the same frame
    (240 of 720 rows, ~10 s of CPU work), scaled to frames/sec."""
    tree = oracle_tree(res["_svo"])
    stride = 3
    secs, n = cpu_frame_sample(tree, res["_fld"], stride, row_offset=stride // 2)
    fps = (n / (WIDTH * HEIGHT)) / secs
    out = {"value": fps, "unit": "frames/s", "cores": os.cpu_count(), "kind": "port",
           "sample": f"oracle render of every {stride}th row ({n} rays) of the 1280x720 frame, {secs:.1f} s"}
    if "_query_pts" in res:
        pts = res["_query_pts"][:: max(1, QUERY_POINTS // 65536)][:65536]
        qs = cpu_query_sample(tree, res["_fld"], pts)
        out["query"] = {"value": len(pts) / qs / 1e6, "unit": "Mpoints/s",
                        "sample": f"{len(pts)} points, forward L=1..5, {qs:.1f} s"}
    if "train" in res:
        secs, npts = cpu_train_sample(tree, res["train"])
        out["train"] = {"value": npts / secs / 1e6, "unit": "Mpoints/s", "cores": 1,
                        "sample": f"{npts // TRAIN_BATCH} Adam steps of batch {TRAIN_BATCH} "
                                  f"(oracle loss_batch + backward + dense Adam, fp64), {secs:.1f} s"}
    return out


def cpu_train_sample(tree, tr, batches: int = 6):
    """Oracle training steps (trainer.py:223-241 restated) on the same field
    and points; bounded to a few batches."""
    from oracle import train_oracle as TO
    fld = tr["_fld"]
    Z = np.array(fld.Z, dtype=np.float64)
    decs = [TO.f64_decoder(d) for d in fld.decoders]
    params = {"Z": Z}
    for i, d in enumerate(decs):
        for nm in ("W1", "b1", "W2", "b2"):
            params[f"decoder{i + 1}.{nm}"] = getattr(d, nm)
    st = TO.Adam.for_params(params)
    act = list(range(1, MAX_LEVEL + 1))
    t0 = time.perf_counter()
    for b in range(batches):
        sl = slice(b * TRAIN_BATCH, (b + 1) * TRAIN_BATCH)
        loss, g, _ = TO._batch_pass(tree, Z, decs, tr["_pts"][sl], tr["_dist"][sl], act)
        gd = {"Z": g.dZ}
        for i, slot in enumerate(g.dec):
            if slot is not None:
                for nm, arr in zip(("W1", "b1", "W2", "b2"), slot):
                    gd[f"decoder{i + 1}.{nm}"] = arr
        TO.adam_step(params, gd, st, 1e-3)
    return time.perf_counter() - t0, batches * TRAIN_BATCH


# ------------------------------------------------------------------ reference arm

def run_reference(args, rank: int, world: int):
    """The reference's CPU algorithm (oracle port; the reference is pure
    Python and not installable on the box) on the host cores, one bounded
    frame sample per step. Rank 0 only."""
    if rank != 0:
        return
    import torch
    torch.cuda.set_device(0)
    knot, svo, fld = build_workload()   # the device build only prepares identical inputs
    tree = oracle_tree(svo)
    stride = 32
    times, rays = [], 0
    for k in range(args.warmup + args.steps):
        secs, n = cpu_frame_sample(tree, fld, stride, row_offset=k % stride)
        if k >= args.warmup:
            times.append(secs)
            rays = n
    ms = statistics.mean(times) * 1e3 * stride  # per full frame
    fps = 1000.0 / ms
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp64", "data": "synthetic (same workload as ours)",
        "config": {"workload": "configs[1]: LOD5 torus-knot octree, 1280x720 sparse sphere trace + normals",
                   "resolution": [WIDTH, HEIGHT]},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": os.cpu_count(), "kind": "port",
                         "sample": f"each step: every {stride}th row ({rays} rays), scaled x{stride}"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
