"""Sparse voxel octree over B = [-1, 1]^3, built and queried on the GPU.

Drop-in for octfield.octree (octree.py:1-357). Same public names, argument
meaning and errors; the structure lives in device memory:

* per traversal level t (levels -log2(r0) .. max_level): sorted Morton
  codes, an occupancy bitmap (one bit per cell, Morton order) with a
  per-word popcount prefix ("rank"), and for t below the finest level the
  first-child index and 8-bit child mask used by the traversal;
* per stored level: parent indices and, for feature levels, the (n, 8)
  global corner-id table.

`build_octree` runs entirely on the device (mark -> closure -> rank ->
extract -> tables); host copies of codes/parents/corners are materialised
lazily when a caller reads them, so a reference user sees the same numpy
fields (OctreeLevel.codes etc.).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream_ptr
from .errors import StructuralError

DOMAIN_MIN = -1.0
DOMAIN_MAX = 1.0
DEFAULT_R0 = 4
_SPAN = DOMAIN_MAX - DOMAIN_MIN

CORNER_OFFSETS = np.array([[j & 1, (j >> 1) & 1, (j >> 2) & 1] for j in range(8)], dtype=np.int64)

# bitmap-backed levels: (2*res)^3 corner bits must stay addressable
_MAX_RES = 2048


def _dev():
    return _lib.device()


def _to_dev_f64(a) -> torch.Tensor:
    t = torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64))
    return t.to(_dev(), non_blocking=False)


def _u64_host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


# ---------------------------------------------------------------- morton

def morton_encode(ijk) -> np.ndarray:
    """Interleave 21-bit coordinates into a 63-bit Z-order code (octree.py:35-49)."""
    arr = np.asarray(ijk)
    single = arr.ndim == 1
    arr = np.atleast_2d(arr)
    if arr.shape[-1] != 3:
        raise StructuralError("morton_encode expects integer triples")
    a64 = arr.astype(np.int64)
    if np.any(a64 < 0) or np.any(a64 >= (1 << 21)):
        raise StructuralError("coordinate does not fit in 21 bits")
    n = len(a64)
    out = torch.empty(n, dtype=torch.int64, device=_dev())
    if n:
        src = torch.as_tensor(np.ascontiguousarray(a64)).to(_dev())
        call("ng_morton_encode", ptr(src), n, ptr(out), stream_ptr())
    codes = _u64_host(out)
    return codes[0] if single else codes


def morton_decode(code) -> np.ndarray:
    """octree.py:73-85."""
    arr = np.asarray(code, dtype=np.uint64)
    single = arr.ndim == 0
    arr = np.atleast_1d(arr)
    n = len(arr)
    out = torch.empty((n, 3), dtype=torch.int64, device=_dev())
    if n:
        src = torch.as_tensor(arr.view(np.int64).copy()).to(_dev())
        call("ng_morton_decode", ptr(src), n, ptr(out), stream_ptr())
    ijk = out.cpu().numpy()
    return ijk[0] if single else ijk


# ---------------------------------------------------------------- structure

@dataclass
class Aabb:
    lo: np.ndarray
    hi: np.ndarray

    def __post_init__(self):
        self.lo = np.asarray(self.lo, dtype=np.float64)
        self.hi = np.asarray(self.hi, dtype=np.float64)
        if np.any(self.lo > self.hi):
            raise StructuralError("Aabb with min > max")


class OctreeLevel:
    """One stored level (octree.py:100-104); numpy views are pulled from the
    device on first access."""

    def __init__(self, codes: torch.Tensor, parents: torch.Tensor, corners: torch.Tensor | None):
        self.d_codes = codes
        self.d_parents = parents
        self.d_corners = corners
        self._codes = self._parents = self._corners = None

    @property
    def codes(self) -> np.ndarray:
        if self._codes is None:
            self._codes = _u64_host(self.d_codes)
        return self._codes

    @property
    def parents(self) -> np.ndarray:
        if self._parents is None:
            self._parents = self.d_parents.cpu().numpy()
        return self._parents

    @property
    def corners(self) -> np.ndarray | None:
        if self.d_corners is None:
            return None
        if self._corners is None:
            self._corners = self.d_corners.cpu().numpy()
        return self._corners


class DeviceOctree:
    """Device tensors per traversal level plus the packed C struct."""

    def __init__(self, r0, max_level, codes, bitmaps, ranks, child_start, child_mask, corners, region_lo,
                 region_hi, half_diag):
        self.r0 = r0
        self.max_level = max_level
        self.n_virtual = int(math.log2(r0))
        self.codes = codes            # per traversal level, int64 views of uint64 codes
        self.bitmaps = bitmaps
        self.ranks = ranks
        self.child_start = child_start
        self.child_mask = child_mask
        self.corners = corners        # per traversal level (None where featureless)
        s = _lib.NgOctree()
        s.r0, s.max_level, s.n_virtual = r0, max_level, self.n_virtual
        s.n_tlevels = len(codes)
        for t in range(len(codes)):
            s.count[t] = codes[t].numel()
            s.codes[t] = ptr(codes[t])
            s.bitmap[t] = ptr(bitmaps[t])
            s.rank[t] = ptr(ranks[t])
            s.child_start[t] = ptr(child_start[t]) if child_start[t] is not None else None
            s.child_mask[t] = ptr(child_mask[t]) if child_mask[t] is not None else None
            s.corners[t] = ptr(corners[t]) if corners[t] is not None else None
        for a in range(3):
            s.region_lo[a] = float(region_lo[a])
            s.region_hi[a] = float(region_hi[a])
        s.half_diag_finest = float(half_diag)
        self.struct = s

    def ref(self):
        import ctypes
        return ctypes.byref(self.struct)


@dataclass
class SparseVoxelOctree:
    """octree.py:107-131, with the device structure attached."""

    r0: int
    max_level: int
    levels: list
    corner_count: int
    corner_offsets: np.ndarray
    region: Aabb
    virtual_codes: list = field(default_factory=list)
    device: DeviceOctree | None = None
    virtual_levels: list = field(default_factory=list, repr=False)   # device-backed virtual levels

    def __post_init__(self):
        # the device build passes device-backed virtual levels; a caller may
        # pass plain code arrays (the reference's constructor, octree.py:107-118)
        if self.virtual_levels and not self.virtual_codes:
            self.virtual_codes = [lv.codes for lv in self.virtual_levels]  # <= 64 codes each

    def resolution(self, level: int) -> int:
        return self.r0 << level

    def voxel_edge(self, level: int) -> float:
        return _SPAN / self.resolution(level)

    def half_diagonal(self, level: int) -> float:
        return 0.5 * np.sqrt(3.0) * self.voxel_edge(level)

    def voxel_count(self, level: int) -> int:
        lv = self.levels[level]
        d = getattr(lv, "d_codes", None)
        return int(d.numel()) if d is not None else len(lv.codes)

    def traversal_codes(self) -> list:
        return self.virtual_codes + [lv.codes for lv in self.levels]


def _level_res(r0: int, level: int) -> int:
    return r0 << level if level >= 0 else r0 >> -level


def _words(res: int) -> int:
    return max(1, (res * res * res + 63) // 64)


def points_to_cells(x: np.ndarray, res: int) -> np.ndarray:
    """Half-open binning (octree.py:134-139). Host utility for callers; the
    device kernels bin with the same fp64 expression."""
    f = (np.asarray(x, dtype=np.float64) - DOMAIN_MIN) * (res / _SPAN)
    return np.clip(np.floor(f).astype(np.int64), 0, res - 1)


def cell_origin(cells: np.ndarray, res: int) -> np.ndarray:
    """octree.py:142-143 (host utility)."""
    return DOMAIN_MIN + np.asarray(cells).astype(np.float64) * (_SPAN / res)


def _corner_lattice(oracle, res: int) -> torch.Tensor:
    """fp32 |d| on the (res+1)^3 corner lattice (octree.py:225-237).

    Oracles that carry a `device_sdf` spec (paper_2101_10994_b200.scenes)
    are evaluated by a CUDA kernel; any other callable is evaluated on the
    host in x-slabs exactly as the reference does and uploaded."""
    n = res + 1
    spec = getattr(oracle, "device_sdf", None)
    if spec is not None:
        kind, params = spec
        prm = _to_dev_f64(np.asarray(params, dtype=np.float64).ravel())
        out = torch.empty(n * n * n, dtype=torch.float32, device=_dev())
        call("ng_sdf_lattice", int(kind), ptr(prm), int(prm.numel()), int(res), ptr(out), stream_ptr())
        return out
    axis = DOMAIN_MIN + np.arange(n) * (_SPAN / res)
    yy, zz = np.meshgrid(axis, axis, indexing="ij")
    plane = np.empty((n * n, 3))
    plane[:, 1] = yy.ravel()
    plane[:, 2] = zz.ravel()
    absd = np.empty((n, n, n), dtype=np.float32)
    for i in range(n):
        plane[:, 0] = axis[i]
        absd[i] = np.abs(oracle(plane)).reshape(n, n).astype(np.float32)
    return torch.from_numpy(absd.ravel()).to(_dev())


def build_octree(oracle, max_level: int, surface_samples: np.ndarray, r0: int = DEFAULT_R0,
                 corner_test: bool = True) -> SparseVoxelOctree:
    """Construct the octree from surface occupancy on the GPU (octree.py:146-222).

    Finest occupancy = cells holding a sample U (oracle and corner_test)
    cells whose minimum corner |d| <= edge*sqrt(2)/2; coarser levels are the
    parent closure; corner ids are level offset + rank of the corner's
    Morton key. Bit-identical to the reference given the same samples and
    |d| lattice.
    """
    if max_level < 1:
        raise StructuralError("max_level must be >= 1")
    if r0 < 2 or (r0 & (r0 - 1)) != 0:
        raise StructuralError("r0 must be a power of two >= 2")
    res = r0 << max_level
    if res >= 1 << 21:
        raise StructuralError("finest resolution exceeds the Morton range")
    if res > _MAX_RES:
        raise StructuralError(f"finest resolution {res} above the device bitmap limit {_MAX_RES}")
    dev = _dev()
    st = stream_ptr()
    samples = np.atleast_2d(np.asarray(surface_samples, dtype=np.float64))
    nv = int(math.log2(r0))
    T = nv + max_level + 1
    resl = [_level_res(r0, t - nv) for t in range(T)]
    bitmaps = [torch.zeros(_words(r), dtype=torch.int64, device=dev) for r in resl]

    if samples.size and len(samples):
        d_s = _to_dev_f64(samples.reshape(-1, 3))
        call("ng_build_mark_samples", ptr(d_s), len(samples), res, ptr(bitmaps[-1]), st)
    if oracle is not None and corner_test:
        tol = (_SPAN / res) * (np.sqrt(2.0) / 2.0)
        absd = _corner_lattice(oracle, res)
        call("ng_build_mark_lattice", ptr(absd), res, float(tol), ptr(bitmaps[-1]), st)
        del absd

    # parent closure up to level 0 and through the virtual grids (octree.py:183-187, 208-212)
    for t in range(T - 1, 0, -1):
        call("ng_bitmap_parent", ptr(bitmaps[t]), bitmaps[t].numel(), ptr(bitmaps[t - 1]),
             bitmaps[t - 1].numel(), st)

    totals = torch.zeros(T + max_level + 1, dtype=torch.int64, device=dev)
    max_words = max(b.numel() for b in bitmaps)
    scratch = torch.empty(_scratch_words(max_words), dtype=torch.int64, device=dev)
    ranks = []
    for t in range(T):
        rk = torch.empty(bitmaps[t].numel(), dtype=torch.int32, device=dev)
        call("ng_bitmap_rank", ptr(bitmaps[t]), bitmaps[t].numel(), ptr(rk), ptr(totals[t:t + 1]),
             ptr(scratch), scratch.numel() * 8, st)
        ranks.append(rk)

    # corner bitmaps per feature level: coordinates 0..res need (2*res)^3 bits
    corner_bm, corner_rk = {}, {}
    counts_host = totals[:T].cpu().numpy()
    if counts_host[-1] == 0:
        raise StructuralError("no occupied voxels; is the surface inside B?")
    codes = []
    for t in range(T):
        c = torch.empty(int(counts_host[t]), dtype=torch.int64, device=dev)
        call("ng_bitmap_extract", ptr(bitmaps[t]), ptr(ranks[t]), bitmaps[t].numel(), ptr(c), st)
        codes.append(c)
    for lv in range(1, max_level + 1):
        t = lv + nv
        cbm = torch.zeros(_words(2 * resl[t]), dtype=torch.int64, device=dev)
        call("ng_corner_mark", ptr(codes[t]), codes[t].numel(), ptr(cbm), st)
        crk = torch.empty(cbm.numel(), dtype=torch.int32, device=dev)
        if _scratch_words(cbm.numel()) > scratch.numel():
            scratch = torch.empty(_scratch_words(cbm.numel()), dtype=torch.int64, device=dev)
        call("ng_bitmap_rank", ptr(cbm), cbm.numel(), ptr(crk), ptr(totals[T + lv:T + lv + 1]), ptr(scratch),
             scratch.numel() * 8, st)
        corner_bm[lv], corner_rk[lv] = cbm, crk
    corner_counts = totals[T:].cpu().numpy()

    parents, child_start, child_mask, corners = [], [], [], []
    offsets = np.zeros(max_level + 1, dtype=np.int64)
    total_corners = 0
    for t in range(T):
        n = codes[t].numel()
        lv = t - nv
        if t + 1 < T:
            cs = torch.empty(n, dtype=torch.int32, device=dev)
            cm = torch.empty(n, dtype=torch.uint8, device=dev)
            call("ng_level_children", ptr(codes[t]), n, ptr(bitmaps[t + 1]), ptr(ranks[t + 1]), ptr(cs),
                 ptr(cm), st)
        else:
            cs = cm = None
        child_start.append(cs)
        child_mask.append(cm)
        if lv >= 1:
            p = torch.empty(n, dtype=torch.int32, device=dev)
            call("ng_level_parents", ptr(codes[t]), n, ptr(bitmaps[t - 1]), ptr(ranks[t - 1]), ptr(p), st)
            ct = torch.empty((n, 8), dtype=torch.int32, device=dev)
            offsets[lv] = total_corners
            call("ng_corner_table", ptr(codes[t]), n, ptr(corner_bm[lv]), ptr(corner_rk[lv]), int(total_corners),
                 ptr(ct), st)
            total_corners += int(corner_counts[lv])
            parents.append(p)
            corners.append(ct)
        elif lv == 0:
            parents.append(torch.full((n,), -1, dtype=torch.int32, device=dev))
            corners.append(None)
        else:
            parents.append(None)
            corners.append(None)
    del corner_bm, corner_rk

    # region AABB of the occupied finest voxels (octree.py:204-206)
    mm = torch.empty(6, dtype=torch.int32, device=dev)
    call("ng_cell_extent", ptr(codes[-1]), codes[-1].numel(), ptr(mm), st)
    mm_h = mm.cpu().numpy().astype(np.int64)
    lo = cell_origin(mm_h[None, :3], res)[0]
    hi = (cell_origin(mm_h[None, 3:], res) + _SPAN / res)[0]
    half_diag = 0.5 * np.sqrt(3.0) * (_SPAN / res)

    dev_tree = DeviceOctree(r0, max_level, codes, bitmaps, ranks, child_start, child_mask, corners, lo, hi,
                            half_diag)
    levels = [OctreeLevel(codes[nv + lv], parents[nv + lv], corners[nv + lv]) for lv in range(max_level + 1)]
    virtual = [OctreeLevel(codes[t], None, None) for t in range(nv)]
    return SparseVoxelOctree(r0=r0, max_level=max_level, levels=levels, corner_count=int(total_corners),
                             corner_offsets=offsets, region=Aabb(lo, hi), virtual_levels=virtual, device=dev_tree)


def octree_from_levels(r0: int, max_level: int, codes: list, parents: list, corners: list, corner_count: int,
                       corner_offsets) -> SparseVoxelOctree:
    """Device octree from stored levels (the model file's topology,
    modelio.py:102-165): occupancy bitmaps from the given codes, the virtual
    grids by parent closure of level 0, ranks and child tables on the device;
    corner tables are taken as stored. The region AABB is recomputed from the
    finest level (modelio.py:95-98)."""
    if len(codes) != max_level + 1:
        raise StructuralError("one code array per stored level is required")
    if (r0 << max_level) > _MAX_RES:
        raise StructuralError(f"finest resolution {r0 << max_level} above the device bitmap limit {_MAX_RES}")
    dev = _dev()
    st = stream_ptr()
    nv = int(math.log2(r0))
    T = nv + max_level + 1
    resl = [_level_res(r0, t - nv) for t in range(T)]
    bitmaps = [None] * T
    for lv in range(max_level + 1):
        c = np.asarray(codes[lv], dtype=np.uint64)
        words = np.zeros(_words(resl[nv + lv]), dtype=np.uint64)
        np.bitwise_or.at(words, (c >> np.uint64(6)).astype(np.int64), np.uint64(1) << (c & np.uint64(63)))
        bitmaps[nv + lv] = torch.from_numpy(words.view(np.int64)).to(dev)
    for t in range(nv - 1, -1, -1):
        bitmaps[t] = torch.zeros(_words(resl[t]), dtype=torch.int64, device=dev)
        call("ng_bitmap_parent", ptr(bitmaps[t + 1]), bitmaps[t + 1].numel(), ptr(bitmaps[t]), bitmaps[t].numel(),
             st)
    totals = torch.zeros(T, dtype=torch.int64, device=dev)
    scratch = torch.empty(_scratch_words(max(b.numel() for b in bitmaps)), dtype=torch.int64, device=dev)
    ranks = []
    for t in range(T):
        rk = torch.empty(bitmaps[t].numel(), dtype=torch.int32, device=dev)
        call("ng_bitmap_rank", ptr(bitmaps[t]), bitmaps[t].numel(), ptr(rk), ptr(totals[t:t + 1]), ptr(scratch),
             scratch.numel() * 8, st)
        ranks.append(rk)
    counts = totals.cpu().numpy()
    d_codes = []
    for t in range(T):
        if t >= nv:
            c = torch.from_numpy(np.ascontiguousarray(np.asarray(codes[t - nv], dtype=np.uint64).view(np.int64)))
            d_codes.append(c.to(dev))
        else:
            c = torch.empty(int(counts[t]), dtype=torch.int64, device=dev)
            call("ng_bitmap_extract", ptr(bitmaps[t]), ptr(ranks[t]), bitmaps[t].numel(), ptr(c), st)
            d_codes.append(c)
    child_start, child_mask, d_parents, d_corners = [], [], [], []
    for t in range(T):
        n = d_codes[t].numel()
        lv = t - nv
        if t + 1 < T:
            cs = torch.empty(n, dtype=torch.int32, device=dev)
            cm = torch.empty(n, dtype=torch.uint8, device=dev)
            call("ng_level_children", ptr(d_codes[t]), n, ptr(bitmaps[t + 1]), ptr(ranks[t + 1]), ptr(cs), ptr(cm),
                 st)
        else:
            cs = cm = None
        child_start.append(cs)
        child_mask.append(cm)
        if lv >= 1:
            d_parents.append(torch.from_numpy(np.ascontiguousarray(parents[lv], dtype=np.int32)).to(dev))
            d_corners.append(torch.from_numpy(np.ascontiguousarray(corners[lv], dtype=np.int32).reshape(-1, 8)).to(dev))
        elif lv == 0:
            d_parents.append(torch.full((n,), -1, dtype=torch.int32, device=dev))
            d_corners.append(None)
        else:
            d_parents.append(None)
            d_corners.append(None)
    res = r0 << max_level
    ijk = morton_decode(np.asarray(codes[max_level], dtype=np.uint64))
    org = cell_origin(ijk, res)
    lo = org.min(axis=0)
    hi = (org + _SPAN / res).max(axis=0)
    half_diag = 0.5 * np.sqrt(3.0) * (_SPAN / res)
    dev_tree = DeviceOctree(r0, max_level, d_codes, bitmaps, ranks, child_start, child_mask, d_corners, lo, hi,
                            half_diag)
    levels = [OctreeLevel(d_codes[nv + lv], d_parents[nv + lv], d_corners[nv + lv]) for lv in range(max_level + 1)]
    virtual = [OctreeLevel(d_codes[t], None, None) for t in range(nv)]
    return SparseVoxelOctree(r0=r0, max_level=max_level, levels=levels, corner_count=int(corner_count),
                             corner_offsets=np.asarray(corner_offsets, dtype=np.int64), region=Aabb(lo, hi),
                             virtual_levels=virtual, device=dev_tree)


def _scratch_words(n_words: int) -> int:
    tiles = (n_words + 2047) // 2048
    return 4 + tiles + 16


# ---------------------------------------------------------------- queries

def _check_domain(pts: np.ndarray) -> None:
    if np.any(pts < DOMAIN_MIN) or np.any(pts > DOMAIN_MAX):
        raise StructuralError("point outside the domain box")


def locate(svo: SparseVoxelOctree, x, level: int) -> np.ndarray:
    """Index of the occupied voxel containing each point, or -1 (octree.py:259-273)."""
    pts = np.asarray(x, dtype=np.float64)
    single = pts.ndim == 1
    pts = np.atleast_2d(pts)
    _check_domain(pts)
    if not 0 <= level <= svo.max_level:
        raise StructuralError(f"level {level} outside 0..{svo.max_level}")
    n = len(pts)
    out = torch.empty(n, dtype=torch.int64, device=_dev())
    if n:
        d = _to_dev_f64(pts)
        call("ng_locate", svo.device.ref(), ptr(d), n, int(level), ptr(out), stream_ptr())
    idx = out.cpu().numpy()
    return idx[0] if single else idx


def locate_device(svo: SparseVoxelOctree, pts: torch.Tensor, level: int) -> torch.Tensor:
    """Zero-copy variant on a (n, 3) float64 CUDA tensor."""
    n = pts.shape[0]
    out = torch.empty(n, dtype=torch.int64, device=pts.device)
    if n:
        pc = pts.contiguous()
        call("ng_locate", svo.device.ref(), ptr(pc), n, int(level), ptr(out), stream_ptr())
    return out


def voxel_bounds(svo: SparseVoxelOctree, level: int, indices) -> tuple:
    """(lo, hi) world bounds of the given voxels (octree.py:285-290)."""
    res = svo.resolution(level)
    idx = torch.as_tensor(np.atleast_1d(np.asarray(indices, dtype=np.int64))).to(_dev())
    codes = svo.levels[level].d_codes.index_select(0, idx)
    out = torch.empty((codes.numel(), 3), dtype=torch.int64, device=_dev())
    if codes.numel():
        call("ng_morton_decode", ptr(codes), codes.numel(), ptr(out), stream_ptr())
    lo = cell_origin(out.cpu().numpy(), res)
    return lo, lo + _SPAN / res


def clamp_into(x: np.ndarray, lo: np.ndarray, hi: np.ndarray) -> np.ndarray:
    """octree.py:293-300 (host utility; the march kernel clamps on device)."""
    return np.clip(x, lo, hi - (hi - lo) * 1e-9)


def children_ranges(parent_codes: np.ndarray, child_codes: np.ndarray):
    """octree.py:303-308 (host utility; the device keeps per-voxel
    child_start / child_mask instead)."""
    base = np.asarray(parent_codes, dtype=np.uint64) << np.uint64(3)
    start = np.searchsorted(child_codes, base)
    end = np.searchsorted(child_codes, base + np.uint64(8))
    return start.astype(np.int64), end.astype(np.int64)


def ray_aabb_batch(origins, dirs, lo, hi):
    """Slab test broadcast over matched rows (octree.py:311-333), on device.
    Returns (t_enter, t_exit, hit)."""
    o, d, l, h = np.broadcast_arrays(np.asarray(origins, dtype=np.float64), np.asarray(dirs, dtype=np.float64),
                                     np.asarray(lo, dtype=np.float64), np.asarray(hi, dtype=np.float64))
    shape = o.shape[:-1]
    flat = [np.ascontiguousarray(a.reshape(-1, 3)) for a in (o, d, l, h)]
    n = len(flat[0])
    te = torch.empty(n, dtype=torch.float64, device=_dev())
    tx = torch.empty(n, dtype=torch.float64, device=_dev())
    hit = torch.empty(n, dtype=torch.uint8, device=_dev())
    if n:
        dv = [_to_dev_f64(a) for a in flat]
        call("ng_ray_aabb", *(ptr(a) for a in dv), n, ptr(te), ptr(tx), ptr(hit), stream_ptr())
    return (te.cpu().numpy().reshape(shape), tx.cpu().numpy().reshape(shape),
            hit.cpu().numpy().astype(bool).reshape(shape))


def ray_aabb(origin, direction, box: Aabb):
    """Single-ray wrapper (octree.py:336-349): (t_enter, t_exit) or None."""
    direction = np.asarray(direction, dtype=np.float64)
    if not direction.any():
        raise StructuralError("ray direction must be nonzero")
    te, tx, hit = ray_aabb_batch(np.asarray(origin, dtype=np.float64)[None, :], direction[None, :],
                                 box.lo[None, :], box.hi[None, :])
    if not hit[0]:
        return None
    return float(te[0]), float(tx[0])


def storage_bytes(svo: SparseVoxelOctree, m: int) -> int:
    """(m + 1) * |V| over feature levels (octree.py:352-357)."""
    return (m + 1) * sum(svo.voxel_count(lv) for lv in range(1, svo.max_level + 1))
