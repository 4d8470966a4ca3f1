"""Breadth-first ray-octree intersection on the GPU (traversal.py:1-275).

All rays descend together one level per pass. Each pass is one kernel that
fuses decide (fp64 slab test + occupied-child count), the exclusive scan
(decoupled look-back) and subdivide (children front to back) -- or, at the
target level, compactify with entry/exit distances. Lists are bit-identical
to the reference's, including order (tests/test_gpu_parity.py::test_traversal_golden_bit_exact;
the render path's lists: tests/test_gpu_render_lists.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream_ptr
from .errors import StructuralError
from .octree import SparseVoxelOctree, cell_origin, ray_aabb_batch

_SPAN = 2.0

# Row d: front-to-back octant order for direction-sign mask d (traversal.py:32-37).
FRONT_TO_BACK = np.array([[k ^ d for k in range(8)] for d in range(8)], dtype=np.int64)


@dataclass
class RayBundle:
    """traversal.py:40-56."""

    origins: np.ndarray
    directions: np.ndarray

    def __post_init__(self):
        self.origins = np.atleast_2d(np.asarray(self.origins, dtype=np.float64))
        self.directions = np.atleast_2d(np.asarray(self.directions, dtype=np.float64))
        if self.origins.shape != self.directions.shape or self.origins.shape[1] != 3:
            raise StructuralError("origins and directions must both be (n, 3)")
        norms = np.linalg.norm(self.directions, axis=1)
        if np.any(np.abs(norms - 1.0) > 1e-6):
            raise StructuralError("ray directions must be unit length")

    @property
    def count(self) -> int:
        return len(self.origins)


@dataclass
class RayVoxelPairList:
    """Pairs at one traversal level (traversal.py:59-70)."""

    level: int
    rays: np.ndarray
    voxels: np.ndarray
    t_enter: np.ndarray | None = None
    t_exit: np.ndarray | None = None

    def __len__(self) -> int:
        return len(self.rays)


def device_rays(rays: RayBundle) -> torch.Tensor:
    """ng_ray records (origin, direction, 1/direction, sign/zero flags)."""
    n = rays.count
    buf = torch.empty(max(n, 1) * _lib.RAY_BYTES, dtype=torch.uint8, device=_lib.device())
    if n:
        o = torch.from_numpy(np.ascontiguousarray(rays.origins)).to(_lib.device())
        d = torch.from_numpy(np.ascontiguousarray(rays.directions)).to(_lib.device())
        call("ng_rays_from_arrays", ptr(o), ptr(d), n, ptr(buf), stream_ptr())
    return buf


def _n_virtual(svo) -> int:
    return svo.device.n_virtual


def _codes_at(svo: SparseVoxelOctree, level: int) -> np.ndarray:
    nv = _n_virtual(svo)
    if level < -nv or level > svo.max_level:
        raise StructuralError(f"no traversal level {level}")
    return svo.virtual_codes[nv + level] if level < 0 else svo.levels[level].codes


def _level_res(svo, level: int) -> int:
    return svo.r0 << level if level >= 0 else svo.r0 >> -level


def pair_bounds(svo: SparseVoxelOctree, pairs: RayVoxelPairList):
    """World AABBs of a pair list's voxels (traversal.py:86-92)."""
    nv = _n_virtual(svo)
    res = _level_res(svo, pairs.level)
    d_codes = svo.device.codes[pairs.level + nv]
    idx = torch.from_numpy(np.ascontiguousarray(pairs.voxels, dtype=np.int64)).to(_lib.device())
    codes = d_codes.index_select(0, idx)
    ijk = torch.empty((codes.numel(), 3), dtype=torch.int64, device=_lib.device())
    if codes.numel():
        call("ng_morton_decode", ptr(codes), codes.numel(), ptr(ijk), stream_ptr())
    lo = cell_origin(np.atleast_2d(ijk.cpu().numpy()), res)
    return lo, lo + _SPAN / res


def _pairs_dev(pairs: RayVoxelPairList) -> torch.Tensor:
    a = np.stack([np.asarray(pairs.rays, dtype=np.int32), np.asarray(pairs.voxels, dtype=np.int32)], axis=1)
    return torch.from_numpy(np.ascontiguousarray(a)).to(_lib.device())


def decide(rays: RayBundle, pairs: RayVoxelPairList, svo: SparseVoxelOctree, final: bool = False) -> np.ndarray:
    """0 on miss, 1 on a final-level hit, else the occupied child count (traversal.py:95-110)."""
    n = len(pairs)
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    t = pairs.level + _n_virtual(svo)
    D = torch.empty(n, dtype=torch.int64, device=_lib.device())
    d_rays, d_pairs = device_rays(rays), _pairs_dev(pairs)  # keep alive until the kernel is enqueued
    call("ng_decide", svo.device.ref(), ptr(d_rays), t, int(bool(final)), ptr(d_pairs), n, ptr(D), stream_ptr())
    return D.cpu().numpy()


def exclusive_sum_serial(d) -> np.ndarray:
    """The serial reference scan S_i = d_0 + ... + d_{i-1} (traversal.py:113-118)."""
    a = np.asarray(d, dtype=np.int64)
    out = np.zeros(len(a), dtype=np.int64)
    np.cumsum(a[:-1], out=out[1:])
    return out


def exclusive_sum_device(d: torch.Tensor) -> torch.Tensor:
    n = d.numel()
    out = torch.empty(n, dtype=torch.int64, device=d.device)
    if n:
        nbytes = _lib.lib().ng_scan_scratch_bytes(n)
        scratch = torch.empty((nbytes + 7) // 8, dtype=torch.int64, device=d.device)
        call("ng_exclusive_sum_i64", ptr(d), n, ptr(out), ptr(scratch), scratch.numel() * 8, stream_ptr())
    return out


def exclusive_sum(d) -> np.ndarray:
    """Single-pass decoupled look-back scan on the device; bit-equal to the
    serial scan (traversal.py:121-144)."""
    a = np.ascontiguousarray(np.asarray(d, dtype=np.int64))
    if len(a) == 0:
        return np.zeros(0, dtype=np.int64)
    return exclusive_sum_device(torch.from_numpy(a).to(_lib.device())).cpu().numpy()


def direction_masks(directions: np.ndarray) -> np.ndarray:
    """Sign octant per ray, bit a set when component a < 0 (traversal.py:147-154)."""
    neg = np.asarray(directions) < 0.0
    return neg[:, 0].astype(np.int64) | (neg[:, 1].astype(np.int64) << 1) | (neg[:, 2].astype(np.int64) << 2)


def ordered_children(direction) -> np.ndarray:
    """traversal.py:157-162."""
    d = np.asarray(direction, dtype=np.float64)
    if not d.any():
        raise StructuralError("ray direction must be nonzero")
    return FRONT_TO_BACK[int(direction_masks(d[None, :])[0])]


def subdivide(pairs: RayVoxelPairList, D: np.ndarray, S: np.ndarray, svo: SparseVoxelOctree,
              rays: RayBundle) -> RayVoxelPairList:
    """Children of hit pairs, front to back per parent (traversal.py:165-191)."""
    D = np.asarray(D, dtype=np.int64)
    S = np.asarray(S, dtype=np.int64)
    total = int(S[-1] + D[-1]) if len(D) else 0
    nxt = pairs.level + 1
    if total == 0:
        z = np.zeros(0, dtype=np.int64)
        return RayVoxelPairList(nxt, z, z.copy())
    t = pairs.level + _n_virtual(svo)
    dev = _lib.device()
    out = torch.empty((total, 2), dtype=torch.int32, device=dev)
    dD = torch.from_numpy(np.ascontiguousarray(D)).to(dev)
    dS = torch.from_numpy(np.ascontiguousarray(S)).to(dev)
    d_rays, d_pairs = device_rays(rays), _pairs_dev(pairs)
    call("ng_subdivide", svo.device.ref(), ptr(d_rays), t, ptr(d_pairs), len(pairs), ptr(dD), ptr(dS), ptr(out),
         stream_ptr())
    o = out.cpu().numpy().astype(np.int64)
    res = RayVoxelPairList(nxt, o[:, 0].copy(), o[:, 1].copy())
    if len(res) != total:
        raise StructuralError("subdivide output size disagrees with the scan")
    return res


def compactify(pairs: RayVoxelPairList, D: np.ndarray, S: np.ndarray) -> RayVoxelPairList:
    """Stable compaction of final-level hits (traversal.py:194-204)."""
    D = np.asarray(D, dtype=np.int64)
    S = np.asarray(S, dtype=np.int64)
    if len(D) and D.max() > 1:
        raise StructuralError("compactify expects final-level decisions in {0, 1}")
    total = int(S[-1] + D[-1]) if len(D) else 0
    if total == 0:
        z = np.zeros(0, dtype=np.int64)
        return RayVoxelPairList(pairs.level, z, z.copy())
    dev = _lib.device()
    out = torch.empty((total, 2), dtype=torch.int32, device=dev)
    dD = torch.from_numpy(np.ascontiguousarray(D)).to(dev)
    dS = torch.from_numpy(np.ascontiguousarray(S)).to(dev)
    d_pairs = _pairs_dev(pairs)
    call("ng_compactify", ptr(d_pairs), len(pairs), ptr(dD), ptr(dS), ptr(out), stream_ptr())
    o = out.cpu().numpy().astype(np.int64)
    return RayVoxelPairList(pairs.level, o[:, 0].copy(), o[:, 1].copy())


class DeviceTrace:
    """Device-resident result of a traversal: every level's pair list plus
    the final hit list (ng_hit_pair records) and its count."""

    def __init__(self, levels, lists, counts, hits, n_hits):
        self.levels = levels      # traversal level tags, coarsest first
        self.lists = lists        # (cap, 2) int32 tensors for intermediate levels (None for root)
        self.counts = counts      # host counts per level
        self.hits = hits          # uint8 buffer of ng_hit_pair records
        self.n_hits = n_hits


def trace_device(rays_dev: torch.Tensor, n: int, svo: SparseVoxelOctree, target: int) -> DeviceTrace:
    """Run the BFS passes with two-phase sizing: counts stay on the device;
    if any list overflowed its capacity the passes rerun with room for it."""
    nv = _n_virtual(svo)
    tt = target + nv
    dev = _lib.device()
    cap = max(8 * n, 4096)
    hit_cap = max(4 * n, 4096)
    while True:
        counts = torch.zeros(tt + 2, dtype=torch.int64, device=dev)
        counts[0] = n
        lists = [None]
        scratch_bytes = _lib.lib().ng_level_scratch_bytes(max(cap, n))
        scratch = torch.empty((scratch_bytes + 7) // 8, dtype=torch.int64, device=dev)
        hits = torch.empty(hit_cap * _lib.HIT_PAIR_BYTES, dtype=torch.uint8, device=dev)
        in_buf, in_cap = None, n
        for t in range(tt):
            out = torch.empty((cap, 2), dtype=torch.int32, device=dev)
            call("ng_traverse_level", svo.device.ref(), ptr(rays_dev), t, 0, ptr(in_buf), ptr(counts[t:t + 1]),
                 in_cap, ptr(out), None, ptr(counts[t + 1:t + 2]), cap, ptr(scratch), scratch.numel() * 8,
                 stream_ptr())
            lists.append(out)
            in_buf, in_cap = out, cap
        call("ng_traverse_level", svo.device.ref(), ptr(rays_dev), tt, 1, ptr(in_buf), ptr(counts[tt:tt + 1]),
             in_cap, None, ptr(hits), ptr(counts[tt + 1:tt + 2]), hit_cap, ptr(scratch), scratch.numel() * 8,
             stream_ptr())
        c = counts.cpu().numpy()
        if c[1:tt + 1].max(initial=0) <= cap and c[tt + 1] <= hit_cap:
            return DeviceTrace(list(range(-nv, target + 1)), lists, c, hits, int(c[tt + 1]))
        cap = max(cap, int(c[1:tt + 1].max(initial=0)) + 1024)
        hit_cap = max(hit_cap, int(c[tt + 1]) + 1024)


def hits_to_numpy(hits: torch.Tensor, n_hits: int):
    raw = hits[:n_hits * _lib.HIT_PAIR_BYTES].cpu().numpy()
    rec = np.frombuffer(raw.tobytes(), dtype=np.dtype([("ray", "<i4"), ("voxel", "<i4"), ("t_enter", "<f8"),
                                                       ("t_exit", "<f8")]))
    return (rec["ray"].astype(np.int64), rec["voxel"].astype(np.int64), rec["t_enter"].copy(),
            rec["t_exit"].copy())


def ray_trace_octree(rays: RayBundle, svo: SparseVoxelOctree, level: int | None = None) -> list:
    """Full descent to `level` (default finest), lists coarsest first
    (traversal.py:207-247): intermediate lists are the candidates entering
    each level; the last holds hits with t_enter / t_exit."""
    target = svo.max_level if level is None else level
    if not 0 <= target <= svo.max_level:
        raise StructuralError(f"target level {target} outside 0..{svo.max_level}")
    n = rays.count
    tr = trace_device(device_rays(rays), n, svo, target)
    nv = _n_virtual(svo)
    out = [RayVoxelPairList(-nv, np.arange(n, dtype=np.int64), np.zeros(n, dtype=np.int64))]
    for i in range(1, len(tr.levels) - 0):
        lvl = tr.levels[i]
        k = int(tr.counts[i])
        a = tr.lists[i][:k].cpu().numpy().astype(np.int64)
        out.append(RayVoxelPairList(lvl, a[:, 0].copy(), a[:, 1].copy()))
    r, v, te, tx = hits_to_numpy(tr.hits, tr.n_hits)
    out[-1] = RayVoxelPairList(target, r, v, te, tx)
    return out


def ray_segments(final: RayVoxelPairList, ray_count: int):
    """Per-ray [start, end) into the final list (traversal.py:250-255)."""
    dev = _lib.device()
    n = len(final)
    start = torch.zeros(ray_count, dtype=torch.int64, device=dev)
    end = torch.zeros(ray_count, dtype=torch.int64, device=dev)
    if ray_count:
        rec = np.zeros(n, dtype=np.dtype([("ray", "<i4"), ("voxel", "<i4"), ("t_enter", "<f8"), ("t_exit", "<f8")]))
        rec["ray"] = final.rays
        rec["voxel"] = final.voxels
        hits = torch.from_numpy(np.frombuffer(rec.tobytes(), dtype=np.uint8).copy()).to(dev) if n else \
            torch.zeros(_lib.HIT_PAIR_BYTES, dtype=torch.uint8, device=dev)
        cnt = torch.tensor([n], dtype=torch.int64, device=dev)
        call("ng_segments", ptr(hits), ptr(cnt), n, ray_count, ptr(start), ptr(end), stream_ptr())
    return start.cpu().numpy(), end.cpu().numpy()


def dump_pairs(path, svo: SparseVoxelOctree, rays: RayBundle, lists) -> None:
    """CSV dump of every pair list: ray, level, morton, t_enter (traversal.py:258-275)."""
    import csv

    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["ray", "level", "morton", "t_enter"])
        for pairs in lists:
            if len(pairs) == 0:
                continue
            codes = _codes_at(svo, pairs.level)
            lo, hi = pair_bounds(svo, pairs)
            t0, _, hit = ray_aabb_batch(rays.origins[pairs.rays], rays.directions[pairs.rays], lo, hi)
            t0 = np.where(hit, t0, np.nan)
            for r, c, t in zip(pairs.rays, codes[pairs.voxels], t0):
                w.writerow([int(r), pairs.level, int(c), f"{t:.9g}"])
