"""The exactness arguments behind the tile traversal's fast child test
(traverse.cu child_hits_ordered / axis_crossings / box_hit_ordered),
checked in numpy float64 against ray_aabb_batch's literal slab test
(octree.py:311-333) on random and lattice-degenerate rays. CPU only."""

import math

import numpy as np


def _slab(o, inv, lo, hi):
    near = far = None
    for a in range(3):
        t1 = (lo[a] - o[a]) * inv[a]
        t2 = (hi[a] - o[a]) * inv[a]
        an, af = min(t1, t2), max(t1, t2)
        near = an if a == 0 else max(near, an)
        far = af if a == 0 else min(far, af)
    return near <= far and far >= 0.0


def _half(a, v):
    lo = (0x55, 0x33, 0x0F)[a]
    return (~lo & 0xFF) if v else lo


def _ordered(q0, q1, q2):
    m = 0xFF
    for a in range(3):
        for b in range(3):
            if a == b:
                continue
            if not q0[a] <= q1[b]:
                m &= ~(_half(a, 0) & _half(b, 0))
            if not q1[a] <= q2[b]:
                m &= ~(_half(a, 1) & _half(b, 1))
            if not q1[a] <= q1[b]:
                m &= ~(_half(a, 1) & _half(b, 0))
        if not q1[a] >= 0.0:
            m &= ~_half(a, 0)
    return m & 0xFF


def _front_to_back(x, dm):
    if dm & 1:
        x = ((x & 0x55) << 1) | ((x >> 1) & 0x55)
    if dm & 2:
        x = ((x & 0x33) << 2) | ((x >> 2) & 0x33)
    if dm & 4:
        x = ((x & 0x0F) << 4) | ((x >> 4) & 0x0F)
    return x


def _rays(rng, n, cres):
    h = 2.0 / cres
    for _ in range(n):
        o = []
        for _a in range(3):
            o.append(-1 + rng.integers(-4, 2 * cres + 5) * h / 2 if rng.random() < 0.3 else rng.uniform(-3, 3))
        if rng.random() < 0.4:  # through a lattice point: ties on many planes
            tgt = [-1 + rng.integers(0, cres + 1) * h for _ in range(3)]
            d = [tgt[a] - o[a] for a in range(3)]
        else:
            d = list(rng.uniform(-1, 1, size=3))
        nrm = math.sqrt(sum(x * x for x in d))
        if nrm == 0.0 or any(x == 0.0 for x in d):
            continue
        yield o, [x / nrm for x in d]


def test_ordered_child_test_equals_slab_tests():
    rng = np.random.default_rng(7)
    checked = 0
    for cres in (2, 8, 64):
        h = 2.0 / cres
        for o, d in _rays(rng, 6000, cres):
            inv = [1.0 / x for x in d]
            pc = [int(rng.integers(0, cres // 2)) for _ in range(3)]
            plo = [-1 + 2 * pc[a] * h for a in range(3)]
            phi = [plo[a] + 2 * h for a in range(3)]
            if not _slab(o, inv, plo, phi):  # children are tested only under a hit parent
                continue
            dm = sum(1 << a for a in range(3) if d[a] < 0)
            ref = 0
            for oct in range(8):
                lo = [plo[a] + ((oct >> a) & 1) * h for a in range(3)]
                hi = [lo[a] + h for a in range(3)]
                ref |= int(_slab(o, inv, lo, hi)) << oct
            q0, q1, q2 = [], [], []
            for a in range(3):  # axis_crossings: faces and mid plane in ray order
                neg = (dm >> a) & 1
                pf = (2 * pc[a] + (2 if neg else 0) - cres // 2) * h
                hs = -h if neg else h
                pm, pl = pf + hs, pf + 2 * hs
                q0.append((pf - o[a]) * inv[a])
                q1.append((pm - o[a]) * inv[a])
                q2.append((pl - o[a]) * inv[a])
            assert _ordered(q0, q1, q2) == _front_to_back(ref, dm)
            checked += 1
    assert checked > 2000


def test_child_hit_implies_parent_hit_and_region_cull():
    """A box inside another on the same dyadic planes: hitting the inner box
    implies hitting the outer one (the root region cull)."""
    rng = np.random.default_rng(3)
    res = 64
    h = 2.0 / res
    for o, d in _rays(rng, 4000, res):
        inv = [1.0 / x for x in d]
        c = [int(rng.integers(0, res)) for _ in range(3)]
        lo = [-1 + c[a] * h for a in range(3)]
        hi = [lo[a] + h for a in range(3)]
        g = [int(rng.integers(0, 3)) for _ in range(3)]
        olo = [lo[a] - g[a] * h for a in range(3)]
        ohi = [hi[a] + g[a] * h for a in range(3)]
        if _slab(o, inv, lo, hi):
            assert _slab(o, inv, olo, ohi)
