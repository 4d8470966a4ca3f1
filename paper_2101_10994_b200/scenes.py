"""Synthetic shapes and fields for the parity cases and the benchmark.

Host-side ground truth, as in the reference (geometry.py:141-149 analytic
primitives, sampling.py surface samplers), plus the (2,3) torus knot of
SURVEY.md Appendix A. Each shape is a callable SDF (numpy, float64) that
`build_octree` accepts like a reference oracle; it also carries a
`device_sdf` spec so the octree build evaluates the corner lattice with a
CUDA kernel instead of on the host.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream_ptr
from .field import NeuralField, new_field
from .octree import CORNER_OFFSETS, SparseVoxelOctree, morton_decode

SDF_SPHERE = 1
SDF_TORUS = 2
SDF_POLYLINE = 3


class Shape:
    """SDF oracle with a host evaluator and a device spec."""

    kind = "analytic"

    def __init__(self, name: str, device_kind: int, params):
        self.name = name
        self.device_sdf = (device_kind, np.asarray(params, dtype=np.float64))

    def __call__(self, pts) -> np.ndarray:
        raise NotImplementedError

    def device_eval(self, pts: torch.Tensor) -> torch.Tensor:
        """SDF at (n, 3) float64 CUDA points with the device kernel."""
        kind, params = self.device_sdf
        prm = torch.from_numpy(params).to(_lib.device())
        out = torch.empty(pts.shape[0], dtype=torch.float64, device=pts.device)
        if pts.shape[0]:
            pc = pts.contiguous()
            call("ng_sdf_eval", int(kind), ptr(prm), int(prm.numel()), ptr(pc), pts.shape[0], ptr(out),
                 stream_ptr())
        return out


class Sphere(Shape):
    def __init__(self, radius: float):
        super().__init__("sphere", SDF_SPHERE, [radius])
        self.radius = float(radius)

    def __call__(self, pts):
        return np.linalg.norm(np.atleast_2d(pts), axis=-1) - self.radius


class Torus(Shape):
    """Torus around the y axis (geometry.py:92-94, 145-148)."""

    def __init__(self, major: float, minor: float):
        super().__init__("torus", SDF_TORUS, [major, minor])
        self.major, self.minor = float(major), float(minor)

    def __call__(self, pts):
        p = np.atleast_2d(pts)
        ring = np.hypot(p[:, 0], p[:, 2]) - self.major
        return np.hypot(ring, p[:, 1]) - self.minor


def knot_vertices(segments: int = 1024, p: int = 2, q: int = 3, R: float = 0.5, r: float = 0.2,
                  scale: float = 1.2) -> np.ndarray:
    """(p, q) torus-knot polyline."""
    t = np.arange(segments) * (2.0 * np.pi / segments)
    rho = R + r * np.cos(q * t)
    return np.stack([rho * np.cos(p * t), r * np.sin(q * t), rho * np.sin(p * t)], axis=1) * scale


class PolylineTube(Shape):
    """Distance to a closed polyline minus a tube radius (1-Lipschitz)."""

    def __init__(self, verts: np.ndarray, tube: float, name: str = "polyline"):
        verts = np.asarray(verts, dtype=np.float64)
        super().__init__(name, SDF_POLYLINE, np.concatenate([[tube], verts.ravel()]))
        self.verts = verts
        self.tube = float(tube)

    def __call__(self, pts, chunk: int = 2048):
        pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
        a = self.verts
        ab = np.roll(a, -1, axis=0) - a
        ab2 = np.einsum("ij,ij->i", ab, ab)
        out = np.empty(len(pts))
        for s in range(0, len(pts), chunk):
            p = pts[s:s + chunk]
            ap = p[:, None, :] - a[None]
            h = np.clip(np.einsum("kij,ij->ki", ap, ab) / ab2[None], 0.0, 1.0)
            diff = ap - h[:, :, None] * ab[None]
            out[s:s + chunk] = np.sqrt(np.einsum("kij,kij->ki", diff, diff).min(axis=1)) - self.tube
        return out


def torus_knot(segments: int = 1024, tube: float = 0.08) -> PolylineTube:
    return PolylineTube(knot_vertices(segments), tube, name="torus-knot")


def knot_samples(shape: PolylineTube, count: int, seed: int = 0) -> np.ndarray:
    """Surface samples P[u] + tube * v, v uniform on the sphere."""
    rng = np.random.default_rng(seed)
    u = rng.integers(0, len(shape.verts), size=count)
    v = rng.standard_normal((count, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return shape.verts[u] + shape.tube * v


def sphere_samples(radius: float, count: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    d = rng.standard_normal((count, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return radius * d


def corner_positions(svo: SparseVoxelOctree, level: int) -> np.ndarray:
    """World positions of every voxel corner at a level, (n*8, 3)."""
    res = svo.resolution(level)
    ijk = morton_decode(svo.levels[level].codes)
    return (-1.0 + (ijk[:, None, :] + CORNER_OFFSETS[None]) * (2.0 / res)).reshape(-1, 3)


def planted_field(svo: SparseVoxelOctree, shape, seed: int = 0, device_sdf: bool = True) -> NeuralField:
    """Deterministic field whose level-L decoder reads the true SDF from
    feature channel L-1 at level-L corners: a render
    workload with realistic iteration counts without any training."""
    fld = new_field(svo, seed=seed)
    Z = fld.Z
    decs = fld.decoders
    for L in range(1, svo.max_level + 1):
        pos = corner_positions(svo, L)
        if device_sdf and isinstance(shape, Shape):
            d = shape.device_eval(torch.from_numpy(np.ascontiguousarray(pos)).to(_lib.device())).cpu().numpy()
        else:
            d = np.asarray(shape(pos))
        Z[svo.levels[L].corners.ravel(), L - 1] = d.astype(np.float32)
        dd = decs[L - 1]
        dd.W1[0:2, :] = 0.0
        dd.b1[0:2] = 0.0
        dd.W1[0, 3 + L - 1] = 1.0
        dd.W1[1, 3 + L - 1] = -1.0
        dd.W2[:] = 0.0
        dd.W2[0, 0] = 1.0
        dd.W2[0, 1] = -1.0
        dd.b2[:] = 0.0
    return NeuralField(svo, Z, decs)
