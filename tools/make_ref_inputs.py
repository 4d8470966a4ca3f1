"""Inputs of the reference arm (`bench.py --impl reference`), made by the
REAL reference package.

Run once in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tools/make_ref_inputs.py

It imports `octfield` from /root/reference/pkg/src and
1. builds the configs[1] octree with the reference's `build_octree`
   (octree.py:146-256, corner test on) over the (2,3) torus-knot polyline
   oracle of SURVEY.md Appendix A, 2^17 surface samples, seed 0, L = 5;
2. plants the field (Appendix A) with the reference's `new_field(svo, 0)`:
   channel L-1 of every level-L corner row holds the knot SDF at the corner;
3. writes `bench_data/knot_l5_ref.npz`: the finest level's Morton codes
   (72,125) and the planted channel value of every corner row (117,197 fp32).

The reference arm rebuilds the identical octree from the finest codes with
the reference's own `build_octree(None, 5, finest voxel centres,
corner_test=False)` in about a second (the coarse levels are the parent
closure of the finest occupancy and the corner tables depend on the
occupancy alone); this script checks that rebuild against the full build
level by level. The full build spends ~5 minutes in the oracle's corner
lattice, which is why the box does not repeat it.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "bench_data", "knot_l5_ref.npz")
sys.path.insert(0, REF)

from octfield import field as F  # noqa: E402
from octfield import octree as OT  # noqa: E402


def knot_vertices(segments=1024, p=2, q=3, R=0.5, r=0.2, scale=1.2):
    """SURVEY.md Appendix A."""
    t = np.arange(segments) * (2.0 * np.pi / segments)
    rho = R + r * np.cos(q * t)
    return np.stack([rho * np.cos(p * t), r * np.sin(q * t), rho * np.sin(p * t)], axis=1) * scale


class KnotOracle:
    """Duck-typed reference oracle (octree.py:237 calls oracle(points)):
    distance to the closed polyline minus the tube radius."""

    def __init__(self, verts, tube=0.08):
        self.a = np.asarray(verts, dtype=np.float64)
        self.ab = np.roll(self.a, -1, axis=0) - self.a
        self.ab2 = np.einsum("ij,ij->i", self.ab, self.ab)
        self.tube = tube

    def __call__(self, pts, chunk=2048):
        pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
        out = np.empty(len(pts))
        for s in range(0, len(pts), chunk):
            p = pts[s:s + chunk]
            ap = p[:, None, :] - self.a[None]
            h = np.clip(np.einsum("kij,ij->ki", ap, self.ab) / self.ab2[None], 0.0, 1.0)
            diff = ap - h[:, :, None] * self.ab[None]
            out[s:s + chunk] = np.sqrt(np.einsum("kij,kij->ki", diff, diff).min(axis=1)) - self.tube
        return out


def knot_samples(verts, tube, count, seed=0):
    rng = np.random.default_rng(seed)
    u = rng.integers(0, len(verts), size=count)
    v = rng.standard_normal((count, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return verts[u] + tube * v


def finest_centres(codes, res):
    ijk = OT.morton_decode(codes)
    return OT.cell_origin(ijk, res) + 0.5 * (2.0 / res)


def rebuild(finest_codes, L, r0=4):
    """What the reference arm does on the box."""
    return OT.build_octree(None, L, finest_centres(finest_codes, r0 << L), r0=r0, corner_test=False)


def main():
    verts = knot_vertices()
    oracle = KnotOracle(verts)
    samples = knot_samples(verts, 0.08, 1 << 17, seed=0)
    t0 = time.time()
    svo = OT.build_octree(oracle, 5, samples)
    print(f"reference build_octree (corner test): {time.time() - t0:.0f} s, voxels "
          f"{[svo.voxel_count(lv) for lv in range(6)]}, corners {svo.corner_count}")
    fin = svo.levels[5].codes
    t0 = time.time()
    again = rebuild(fin, 5)
    print(f"rebuild from the finest codes: {time.time() - t0:.1f} s")
    for lv in range(6):
        a, b = svo.levels[lv], again.levels[lv]
        assert np.array_equal(a.codes, b.codes) and np.array_equal(a.parents, b.parents)
        assert (a.corners is None) == (b.corners is None)
        if a.corners is not None:
            assert np.array_equal(a.corners, b.corners)
    assert svo.corner_count == again.corner_count
    assert np.array_equal(svo.corner_offsets, again.corner_offsets)
    assert np.array_equal(svo.region.lo, again.region.lo) and np.array_equal(svo.region.hi, again.region.hi)
    for a, b in zip(svo.virtual_codes, again.virtual_codes):
        assert np.array_equal(a, b)
    # planted channel values (Appendix A): level-L corner rows hold the SDF at the corner
    planted = np.zeros(svo.corner_count, dtype=np.float32)
    for L in range(1, 6):
        res = svo.resolution(L)
        lv = svo.levels[L]
        pos = (-1.0 + (OT.morton_decode(lv.codes)[:, None, :] + OT.CORNER_OFFSETS[None]) * (2.0 / res)).reshape(-1, 3)
        planted[lv.corners.ravel()] = oracle(pos).astype(np.float32)
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez_compressed(OUT, finest_codes=fin, planted=planted, max_level=np.int64(5), r0=np.int64(4),
                        voxels=np.array([svo.voxel_count(lv) for lv in range(6)]),
                        corner_count=np.int64(svo.corner_count))
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes)")
    _ = F  # new_field is applied on the box (seed 0); nothing of it is stored


if __name__ == "__main__":
    main()
