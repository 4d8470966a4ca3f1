"""CPU oracle for the NGLOD render hot path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference package `octfield`
(arxiv/paper_2101_10994, /root/reference/pkg/src/octfield) for the functions
on the hot path named in SURVEY.md section 8(a). It is the checker the GPU
path is compared against. Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it; the
product package never does.

Parity pinning: `tests/golden/make_golden.py` runs the real reference in the
build container and commits its outputs as fixtures; `tests/test_oracle.py`
checks this restatement against those fixtures (and against the live
reference when /root/reference is importable).

Every function cites the reference file:line it restates. Arithmetic is
float64 throughout with the same operation order as the reference so that
integer results (codes, indices, pair lists) are bit-identical.

One deliberate difference: the sphere-trace advance loop is per ray. The
reference's vectorised loop (render.py:202-238) lets one ray's "sliver" skip
re-run the far-plane test for other rays in the same batch; per-ray semantics
equal the reference whenever no voxel is entered beyond the far plane.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

DMIN = -1.0          # geometry.py:24
DMAX = 1.0           # geometry.py:25
SPAN = DMAX - DMIN   # octree.py:26

FEAT_DIM = 32        # field.py:25
HID_DIM = 128        # field.py:26
FEAT_SIGMA = 0.01    # field.py:27


class OracleError(Exception):
    """Raised where the reference raises one of its OctfieldError types."""


# --------------------------------------------------------------------------
# Morton codes (octree.py:35-85). Restated with a per-byte lookup table:
# each input byte spreads to 24 output bits, three bits apart.

_SPREAD8 = np.zeros(256, dtype=np.uint64)
for _b in range(256):
    _v = 0
    for _i in range(8):
        _v |= ((_b >> _i) & 1) << (3 * _i)
    _SPREAD8[_b] = _v
_COMPACT_BITS = [np.uint64(1) << np.uint64(3 * i) for i in range(21)]


def spread_bits(v: np.ndarray) -> np.ndarray:
    v = np.asarray(v, dtype=np.uint64) & np.uint64(0x1FFFFF)
    out = _SPREAD8[(v & np.uint64(0xFF)).astype(np.int64)]
    out = out | (_SPREAD8[((v >> np.uint64(8)) & np.uint64(0xFF)).astype(np.int64)] << np.uint64(24))
    out = out | (_SPREAD8[((v >> np.uint64(16)) & np.uint64(0xFF)).astype(np.int64)] << np.uint64(48))
    return out


def compact_bits(c: np.ndarray) -> np.ndarray:
    c = np.asarray(c, dtype=np.uint64)
    out = np.zeros(c.shape, dtype=np.uint64)
    for i, bit in enumerate(_COMPACT_BITS):
        out |= ((c & bit) >> np.uint64(2 * i))
    return out


def morton_encode(ijk) -> np.ndarray:
    """octree.py:35-49 -- x in bit 0, y in bit 1, z in bit 2 of each triad."""
    a = np.atleast_2d(np.asarray(ijk))
    if a.shape[-1] != 3:
        raise OracleError("morton_encode expects integer triples")
    if np.any(a.astype(np.int64) < 0) or np.any(a.astype(np.int64) >= (1 << 21)):
        raise OracleError("coordinate does not fit in 21 bits")
    a = a.astype(np.uint64)
    return spread_bits(a[:, 0]) | (spread_bits(a[:, 1]) << np.uint64(1)) | (
        spread_bits(a[:, 2]) << np.uint64(2))


def morton_decode(codes) -> np.ndarray:
    """octree.py:73-85."""
    c = np.atleast_1d(np.asarray(codes, dtype=np.uint64))
    return np.stack([compact_bits(c), compact_bits(c >> np.uint64(1)),
                     compact_bits(c >> np.uint64(2))], axis=-1).astype(np.int64)


# --------------------------------------------------------------------------
# Binning (octree.py:134-143)

def bin_points(x, res: int) -> np.ndarray:
    """Half-open binning, clipped into the grid (octree.py:134-139)."""
    f = (np.asarray(x, dtype=np.float64) - DMIN) * (res / SPAN)
    return np.clip(np.floor(f).astype(np.int64), 0, res - 1)


def cell_lo(cells, res: int) -> np.ndarray:
    """World position of a cell's low corner (octree.py:142-143)."""
    return DMIN + np.asarray(cells).astype(np.float64) * (SPAN / res)


# --------------------------------------------------------------------------
# Octree (octree.py:100-131, 146-256)

CORNER_OFS = np.array([[j & 1, (j >> 1) & 1, (j >> 2) & 1] for j in range(8)], dtype=np.int64)


@dataclass
class OracleOctree:
    r0: int
    max_level: int
    codes: list            # per stored level: sorted uint64 codes
    parents: list          # per stored level: int32 parent index (-1 at level 0)
    corners: list          # per stored level: (n, 8) int32 global corner ids (None at 0)
    corner_offsets: np.ndarray
    corner_count: int
    region_lo: np.ndarray
    region_hi: np.ndarray
    virtual_codes: list = field(default_factory=list)

    def res(self, level: int) -> int:
        return self.r0 << level if level >= 0 else self.r0 >> -level

    def edge(self, level: int) -> float:
        return SPAN / self.res(level)

    def half_diag(self, level: int) -> float:
        return 0.5 * np.sqrt(3.0) * self.edge(level)

    def level_codes(self, level: int) -> np.ndarray:
        """Stored or virtual level codes (traversal.py:73-79)."""
        nv = len(self.virtual_codes)
        if level < -nv or level > self.max_level:
            raise OracleError(f"no traversal level {level}")
        return self.virtual_codes[nv + level] if level < 0 else self.codes[level]


def lattice_min_abs(absd: np.ndarray, res: int) -> np.ndarray:
    """Per-cell minimum over the 8 corner |d| values (octree.py:238-242)."""
    m = absd[:res, :res, :res]
    for o in CORNER_OFS[1:]:
        m = np.minimum(m, absd[o[0]:o[0] + res, o[1]:o[1] + res, o[2]:o[2] + res])
    return m


def corner_lattice_absd(sdf, res: int) -> np.ndarray:
    """|d| on the (res+1)^3 corner lattice, rounded to float32, evaluated in
    x-slabs (octree.py:225-237)."""
    n = res + 1
    ax = DMIN + np.arange(n) * (SPAN / res)
    yy, zz = np.meshgrid(ax, ax, indexing="ij")
    plane = np.empty((n * n, 3))
    plane[:, 1] = yy.ravel()
    plane[:, 2] = zz.ravel()
    out = np.empty((n, n, n), dtype=np.float32)
    for i in range(n):
        plane[:, 0] = ax[i]
        out[i] = np.abs(sdf(plane)).reshape(n, n).astype(np.float32)
    return out


def build(sdf, max_level: int, samples, r0: int = 4, corner_test: bool = True,
          absd_lattice: np.ndarray | None = None) -> OracleOctree:
    """build_octree (octree.py:146-222).

    Finest occupancy = binned samples U cells whose min corner |d| (fp32)
    <= edge*sqrt(2)/2 (compared in fp64); coarser levels are the parent
    closure; corner ids are offset + rank among the level's unique corner
    codes (octree.py:249-256). `absd_lattice` lets a caller supply the
    fp32 |d| lattice directly instead of an sdf callable.
    """
    if max_level < 1:
        raise OracleError("max_level must be >= 1")
    if r0 < 2 or (r0 & (r0 - 1)):
        raise OracleError("r0 must be a power of two >= 2")
    res = r0 << max_level
    if res >= 1 << 21:
        raise OracleError("finest resolution exceeds the Morton range")
    pts = np.atleast_2d(np.asarray(samples, dtype=np.float64))
    occupied = np.zeros(0, dtype=np.uint64)
    if len(pts):
        occupied = np.unique(morton_encode(bin_points(pts, res)))
    if corner_test and (sdf is not None or absd_lattice is not None):
        tol = (SPAN / res) * (np.sqrt(2.0) / 2.0)
        absd = absd_lattice if absd_lattice is not None else corner_lattice_absd(sdf, res)
        near = np.argwhere(lattice_min_abs(absd, res) <= tol)
        if len(near):
            occupied = np.union1d(occupied, morton_encode(near))
    if len(occupied) == 0:
        raise OracleError("no occupied voxels")

    per_level = [occupied]
    for _ in range(max_level):
        per_level.insert(0, np.unique(per_level[0] >> np.uint64(3)))

    parents, corners = [], []
    offsets = np.zeros(max_level + 1, dtype=np.int64)
    total = 0
    for lv, codes in enumerate(per_level):
        if lv == 0:
            parents.append(np.full(len(codes), -1, dtype=np.int32))
            corners.append(None)
            continue
        parents.append(np.searchsorted(per_level[lv - 1], codes >> np.uint64(3)).astype(np.int32))
        keys = morton_encode((morton_decode(codes)[:, None, :] + CORNER_OFS[None]).reshape(-1, 3))
        uniq, inv = np.unique(keys, return_inverse=True)
        offsets[lv] = total
        corners.append((inv.reshape(-1, 8) + total).astype(np.int32))
        total += len(uniq)

    fine_lo = cell_lo(morton_decode(per_level[-1]), res)
    region_lo = fine_lo.min(axis=0)
    region_hi = (fine_lo + SPAN / res).max(axis=0)
    nv = int(np.log2(r0))
    virtual = [np.unique(per_level[0] >> np.uint64(3 * (nv - s))) for s in range(nv)]
    return OracleOctree(r0, max_level, per_level, parents, corners, offsets, total,
                        region_lo, region_hi, virtual)


def lookup(sorted_codes: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """Index of each code in a sorted list, -1 if absent (octree.py:276-282)."""
    if len(sorted_codes) == 0:
        return np.full(len(codes), -1, dtype=np.int64)
    pos = np.minimum(np.searchsorted(sorted_codes, codes), len(sorted_codes) - 1)
    return np.where(sorted_codes[pos] == codes, pos, -1).astype(np.int64)


def locate(tree: OracleOctree, x, level: int) -> np.ndarray:
    """octree.py:259-273."""
    p = np.atleast_2d(np.asarray(x, dtype=np.float64))
    if np.any(p < DMIN) or np.any(p > DMAX):
        raise OracleError("point outside the domain box")
    return lookup(tree.codes[level], morton_encode(bin_points(p, tree.res(level))))


def child_range(parent_codes, child_codes):
    """octree.py:303-308."""
    base = np.asarray(parent_codes, dtype=np.uint64) << np.uint64(3)
    return (np.searchsorted(child_codes, base).astype(np.int64),
            np.searchsorted(child_codes, base + np.uint64(8)).astype(np.int64))


def slab(o, d, lo, hi):
    """Closed-box slab test with zero-direction handling (octree.py:311-333).
    Returns (t_enter clamped at 0, t_exit, hit)."""
    o = np.asarray(o, dtype=np.float64)
    d = np.asarray(d, dtype=np.float64)
    zero = d == 0.0
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        ta = (lo - o) * inv
        tb = (hi - o) * inv
    inside = (o >= lo) & (o <= hi)
    lo_t = np.where(zero, np.where(inside, -np.inf, np.inf), np.minimum(ta, tb))
    hi_t = np.where(zero, np.where(inside, np.inf, -np.inf), np.maximum(ta, tb))
    near = lo_t.max(axis=-1)
    far = hi_t.min(axis=-1)
    return np.maximum(near, 0.0), far, (near <= far) & (far >= 0.0)


# --------------------------------------------------------------------------
# Traversal (traversal.py:95-255)

def exclusive_scan(d) -> np.ndarray:
    """traversal.py:113-144 (integer scan; any order is bit-equal)."""
    a = np.asarray(d, dtype=np.int64)
    out = np.zeros(len(a), dtype=np.int64)
    if len(a) > 1:
        np.cumsum(a[:-1], out=out[1:])
    return out


def dir_masks(dirs) -> np.ndarray:
    """Sign octant, bit a set when component a < 0 (traversal.py:147-154)."""
    n = np.asarray(dirs) < 0.0
    return n[:, 0].astype(np.int64) | (n[:, 1].astype(np.int64) << 1) | (n[:, 2].astype(np.int64) << 2)


def voxel_boxes(tree: OracleOctree, level: int, vox):
    """traversal.py:86-92."""
    res = tree.res(level)
    lo = cell_lo(np.atleast_2d(morton_decode(tree.level_codes(level)[vox])), res)
    return lo, lo + SPAN / res


@dataclass
class PairList:
    level: int
    rays: np.ndarray
    voxels: np.ndarray
    t_enter: np.ndarray | None = None
    t_exit: np.ndarray | None = None

    def __len__(self):
        return len(self.rays)


TIE_REL = 2.0 ** -22  # a slab decision this close to flipping would flip in fp32 (SURVEY.md 8c probe)


def count_near_ties(o, d, lo, hi, rel: float = TIE_REL) -> int:
    """Slab decisions (octree.py:311-333) within `rel` of flipping: the hit
    test is max(near) <= min(far) and min(far) >= 0; a decision is a near
    tie when either comparison's two sides differ by at most rel * max(1,
    |side|). These are the pairs a lower-precision slab test could get
    wrong; an exact restatement must still agree on every one of them."""
    o = np.asarray(o, dtype=np.float64)
    d = np.asarray(d, dtype=np.float64)
    zero = d == 0.0
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        ta = (lo - o) * inv
        tb = (hi - o) * inv
        inside = (o >= lo) & (o <= hi)
        near = np.where(zero, np.where(inside, -np.inf, np.inf), np.minimum(ta, tb)).max(axis=-1)
        far = np.where(zero, np.where(inside, np.inf, -np.inf), np.maximum(ta, tb)).min(axis=-1)
        scale = np.maximum(1.0, np.maximum(np.abs(near), np.abs(far)))
        t1 = np.isfinite(near) & np.isfinite(far) & (np.abs(far - near) <= rel * scale)
        t2 = np.isfinite(far) & (np.abs(far) <= rel)
    return int(np.count_nonzero(t1 | t2))


def decide(tree, origins, dirs, pairs: PairList, final: bool, ties: list | None = None) -> np.ndarray:
    """traversal.py:95-110. With `ties`, appends the level's (near-tie
    decisions (count_near_ties), decisions) -- diagnostics only, the
    decisions are unchanged."""
    if len(pairs) == 0:
        if ties is not None:
            ties.append((0, 0))
        return np.zeros(0, dtype=np.int64)
    lo, hi = voxel_boxes(tree, pairs.level, pairs.voxels)
    _, _, hit = slab(origins[pairs.rays], dirs[pairs.rays], lo, hi)
    if ties is not None:
        ties.append((count_near_ties(origins[pairs.rays], dirs[pairs.rays], lo, hi), len(pairs)))
    if final:
        return hit.astype(np.int64)
    s, e = child_range(tree.level_codes(pairs.level)[pairs.voxels],
                       tree.level_codes(pairs.level + 1))
    return np.where(hit, e - s, 0)


def expand(tree, dirs, pairs: PairList, D, S) -> PairList:
    """subdivide (traversal.py:165-191): children of hit pairs, each parent
    block in front-to-back octant order for its ray."""
    nxt = pairs.level + 1
    total = int(S[-1] + D[-1]) if len(D) else 0
    if total == 0:
        z = np.zeros(0, dtype=np.int64)
        return PairList(nxt, z, z.copy())
    keep = np.flatnonzero(D > 0)
    cnt = D[keep]
    child_codes = tree.level_codes(nxt)
    first, _ = child_range(tree.level_codes(pairs.level)[pairs.voxels[keep]], child_codes)
    block = np.repeat(np.arange(len(keep)), cnt)
    child = np.repeat(first, cnt) + (np.arange(total) - np.repeat(S[keep], cnt))
    ray = np.repeat(pairs.rays[keep], cnt)
    key = (child_codes[child] & np.uint64(7)).astype(np.int64) ^ dir_masks(dirs)[ray]
    order = np.lexsort((key, block))
    return PairList(nxt, ray[order], child[order])


def compact(pairs: PairList, D, S) -> PairList:
    """compactify (traversal.py:194-204)."""
    if len(D) and D.max() > 1:
        raise OracleError("compact expects decisions in {0, 1}")
    keep = np.flatnonzero(D == 1)
    return PairList(pairs.level, pairs.rays[keep].astype(np.int64), pairs.voxels[keep].astype(np.int64))


def traverse(tree: OracleOctree, origins, dirs, level: int | None = None, ties: list | None = None) -> list:
    """ray_trace_octree (traversal.py:207-247): lists from the virtual root
    to `level`; intermediate lists are unfiltered candidates, the last holds
    hits with t_enter/t_exit. With `ties` (a list), every level's (near-tie
    decisions, decisions) is appended to it (count_near_ties)."""
    target = tree.max_level if level is None else level
    if not 0 <= target <= tree.max_level:
        raise OracleError(f"target level {target} outside 0..{tree.max_level}")
    origins = np.atleast_2d(np.asarray(origins, dtype=np.float64))
    dirs = np.atleast_2d(np.asarray(dirs, dtype=np.float64))
    n = len(origins)
    cur = PairList(-len(tree.virtual_codes), np.arange(n, dtype=np.int64), np.zeros(n, dtype=np.int64))
    lists = [cur]
    while cur.level < target:
        D = decide(tree, origins, dirs, cur, False, ties)
        cur = expand(tree, dirs, cur, D, exclusive_scan(D))
        lists.append(cur)
    D = decide(tree, origins, dirs, cur, True, ties)
    fin = compact(cur, D, exclusive_scan(D))
    if len(fin):
        lo, hi = voxel_boxes(tree, fin.level, fin.voxels)
        fin.t_enter, fin.t_exit, _ = slab(origins[fin.rays], dirs[fin.rays], lo, hi)
    else:
        fin.t_enter, fin.t_exit = np.zeros(0), np.zeros(0)
    lists[-1] = fin
    return lists


def compare_final_lists(tree: OracleOctree, origins, dirs, got_rays, got_voxels, got_t_enter, got_t_exit,
                        ray_ids, level: int) -> dict:
    """Check a final (ray, voxel, t_enter, t_exit) list produced elsewhere
    against traverse() on the rays `ray_ids` (indices into origins/dirs),
    bit for bit and in order (ray_trace_octree's last list,
    traversal.py:207-247). `got_*` may hold other rays too; only the
    entries of `ray_ids` are compared. Returns pairs compared, the rays whose
    sub-lists differ, how many of those have a near-tie slab decision
    (count_near_ties) and the near-tie decisions of the whole sample."""
    ray_ids = np.asarray(ray_ids, dtype=np.int64)
    ties: list = []
    fin = traverse(tree, origins[ray_ids], dirs[ray_ids], level, ties=ties)[-1]
    got_rays = np.asarray(got_rays, dtype=np.int64)
    pos = np.full(len(origins), -1, dtype=np.int64)
    pos[ray_ids] = np.arange(len(ray_ids))
    sel = pos[got_rays] >= 0
    g_r = pos[got_rays[sel]]
    g_v = np.asarray(got_voxels, dtype=np.int64)[sel]
    g_a = np.asarray(got_t_enter, dtype=np.float64)[sel]
    g_b = np.asarray(got_t_exit, dtype=np.float64)[sel]
    o_r = np.asarray(fin.rays, dtype=np.int64)
    bad = np.zeros(len(ray_ids), dtype=bool)
    if len(g_r) != len(o_r) or not np.array_equal(g_r, o_r):
        gc = np.bincount(g_r, minlength=len(ray_ids))
        oc = np.bincount(o_r, minlength=len(ray_ids))
        bad |= gc != oc
    if not bad.any():
        same = ((g_v == fin.voxels) & (g_a.view(np.int64) == fin.t_enter.view(np.int64))
                & (g_b.view(np.int64) == fin.t_exit.view(np.int64)))
        bad[o_r[~same]] = True
    else:  # compare the rays whose counts agree entry by entry
        for r in np.flatnonzero(~bad):
            gm, om = g_r == r, o_r == r
            if not (np.array_equal(g_v[gm], fin.voxels[om]) and np.array_equal(g_a[gm], fin.t_enter[om])
                    and np.array_equal(g_b[gm], fin.t_exit[om])):
                bad[r] = True
    bad_ids = ray_ids[bad]
    tie_bad = 0
    for r in bad_ids[:1000]:
        t1: list = []
        traverse(tree, origins[r:r + 1], dirs[r:r + 1], level, ties=t1)
        tie_bad += int(sum(a for a, _ in t1) > 0)
    return {"rays": int(len(ray_ids)), "pairs": int(len(o_r)), "mismatched_rays": int(bad.sum()),
            "mismatched_near_tie": tie_bad, "near_tie_decisions": int(sum(a for a, _ in ties)),
            "decisions": int(sum(b for _, b in ties)), "tie_rel": TIE_REL,
            "first_mismatch": int(bad_ids[0]) if len(bad_ids) else None}


def segments(final: PairList, n_rays: int):
    """ray_segments (traversal.py:250-255)."""
    r = np.arange(n_rays, dtype=np.int64)
    return (np.searchsorted(final.rays, r, side="left"),
            np.searchsorted(final.rays, r, side="right"))


# --------------------------------------------------------------------------
# Field (field.py:51-239, 337-357)

@dataclass
class OracleDecoder:
    W1: np.ndarray   # (h, 3 + m) float32
    b1: np.ndarray   # (h,)
    W2: np.ndarray   # (1, h)
    b2: np.ndarray   # (1,)


def init_features(corner_count: int, m: int = FEAT_DIM, seed: int = 0) -> np.ndarray:
    """field.py:51-56."""
    g = np.random.default_rng(seed)
    return (FEAT_SIGMA * g.standard_normal((corner_count, m))).astype(np.float32)


def init_decoders(max_level: int, m: int = FEAT_DIM, h: int = HID_DIM, seed: int = 0) -> list:
    """field.py:59-76 (same RNG draw order)."""
    g = np.random.default_rng(seed)
    k1 = 1.0 / np.sqrt(3 + m)
    k2 = 1.0 / np.sqrt(h)
    out = []
    for _ in range(max_level):
        W1 = g.uniform(-k1, k1, size=(h, 3 + m)).astype(np.float32)
        b1 = g.uniform(-k1, k1, size=h).astype(np.float32)
        W2 = g.uniform(-k2, k2, size=(1, h)).astype(np.float32)
        b2 = g.uniform(-k2, k2, size=1).astype(np.float32)
        out.append(OracleDecoder(W1, b1, W2, b2))
    return out


def new_field(tree: OracleOctree, m: int = FEAT_DIM, h: int = HID_DIM, seed: int = 0):
    """field.py:272-283: features with `seed`, decoders with `seed + 1`."""
    return init_features(tree.corner_count, m, seed), init_decoders(tree.max_level, m, h, seed + 1)


def tri_weights(u: np.ndarray) -> np.ndarray:
    """field.py:122-135 -- corner j weight = wx[j&1] * wy[j>>1&1] * wz[j>>2&1]."""
    wx = np.stack([1.0 - u[:, 0], u[:, 0]], axis=1)
    wy = np.stack([1.0 - u[:, 1], u[:, 1]], axis=1)
    wz = np.stack([1.0 - u[:, 2], u[:, 2]], axis=1)
    jx = CORNER_OFS[:, 0]
    jy = CORNER_OFS[:, 1]
    jz = CORNER_OFS[:, 2]
    return wx[:, jx] * wy[:, jy] * wz[:, jz]


@dataclass
class LevelRecord:
    level: int
    mask: np.ndarray
    ids: np.ndarray
    w: np.ndarray
    psi: np.ndarray


def interp(tree: OracleOctree, Z, pts, level: int) -> LevelRecord:
    """_interp_level (field.py:104-119)."""
    res = tree.res(level)
    idx = locate(tree, pts, level)
    mask = idx >= 0
    psi = np.zeros((len(pts), Z.shape[1]))
    rows = np.flatnonzero(mask)
    if len(rows) == 0:
        return LevelRecord(level, mask, np.zeros((0, 8), np.int32), np.zeros((0, 8)), psi)
    ids = tree.corners[level][idx[rows]]
    cells = morton_decode(tree.codes[level][idx[rows]])
    u = np.clip((pts[rows] - DMIN) * (res / SPAN) - cells, 0.0, 1.0)
    w = tri_weights(u)
    psi[rows] = np.einsum("kj,kjm->km", w, Z[ids].astype(np.float64))
    return LevelRecord(level, mask, ids, w, psi)


def feature_sum(tree, Z, x, L: int):
    """sum_features (field.py:154-169): z = sum of levels 1..L, mask (n, L)."""
    if L < 1:
        raise OracleError("L must be >= 1")
    pts = np.atleast_2d(np.asarray(x, dtype=np.float64))
    z = np.zeros((len(pts), Z.shape[1]))
    mask = np.zeros((len(pts), L), dtype=bool)
    for lv in range(1, L + 1):
        rec = interp(tree, Z, pts, lv)
        z += rec.psi
        mask[:, lv - 1] = rec.mask
    return z, mask


def mlp(dec: OracleDecoder, x, z) -> np.ndarray:
    """decode (field.py:172-182), float64."""
    inp = np.concatenate([np.atleast_2d(np.asarray(x, dtype=np.float64)), np.atleast_2d(z)], axis=1)
    if not np.all(np.isfinite(inp)):
        raise OracleError("non-finite decoder input")
    hid = np.maximum(inp @ dec.W1.T.astype(np.float64) + dec.b1.astype(np.float64), 0.0)
    return (hid @ dec.W2.T.astype(np.float64) + dec.b2.astype(np.float64))[:, 0]


def empty_value(tree: OracleOctree, x) -> np.ndarray:
    """empty_space_value (field.py:185-191)."""
    p = np.atleast_2d(np.asarray(x, dtype=np.float64))
    gap = np.maximum(tree.region_lo - p, 0.0) + np.maximum(p - tree.region_hi, 0.0)
    return np.linalg.norm(gap, axis=1) + tree.half_diag(tree.max_level)


@dataclass
class Counts:
    decoder_evals: int = 0
    evals_missing_level: int = 0
    empty_fallbacks: int = 0


def predict(tree, Z, decoders, x, L: int, counts: Counts | None = None) -> np.ndarray:
    """predict (field.py:194-218)."""
    pts = np.atleast_2d(np.asarray(x, dtype=np.float64))
    if not 1 <= L <= len(decoders):
        raise OracleError(f"level {L} outside 1..{len(decoders)}")
    z, mask = feature_sum(tree, Z, pts, L)
    anyl = mask.any(axis=1)
    out = np.empty(len(pts))
    dec_rows = np.flatnonzero(anyl)
    if len(dec_rows):
        out[dec_rows] = mlp(decoders[L - 1], pts[dec_rows], z[dec_rows])
    miss = np.flatnonzero(~anyl)
    if len(miss):
        out[miss] = empty_value(tree, pts[miss])
    if counts is not None:
        counts.decoder_evals += len(dec_rows)
        counts.evals_missing_level += int((~mask[dec_rows, L - 1]).sum())
        counts.empty_fallbacks += len(miss)
    return out


def blend(tree, Z, decoders, x, lod: float, counts: Counts | None = None) -> np.ndarray:
    """blend (field.py:226-239)."""
    if lod > len(decoders):
        raise OracleError(f"blend level {lod} above max {len(decoders)}")
    lod = max(float(lod), 1.0)
    base = int(np.floor(lod))
    a = lod - base
    if a == 0.0:
        return predict(tree, Z, decoders, x, base, counts)
    lo = predict(tree, Z, decoders, x, base, counts)
    hi = predict(tree, Z, decoders, x, base + 1, counts)
    return (1.0 - a) * lo + a * hi


def forward_levels(tree, Z, decoders, x, levels) -> np.ndarray:
    """Batched SDF query: forward (field.py:337-357) for each L in `levels`,
    one column per level. Levels are interpolated once and prefix-summed;
    the result equals calling forward(x, L) per L."""
    pts = np.atleast_2d(np.asarray(x, dtype=np.float64))
    Lmax = max(levels)
    recs = [interp(tree, Z, pts, lv) for lv in range(1, Lmax + 1)]
    out = np.empty((len(pts), len(levels)))
    for col, L in enumerate(levels):
        z = np.zeros((len(pts), Z.shape[1]))
        anyl = np.zeros(len(pts), dtype=bool)
        for r in recs[:L]:
            z += r.psi
            anyl |= r.mask
        rows = np.flatnonzero(anyl)
        if len(rows):
            out[rows, col] = mlp(decoders[L - 1], pts[rows], z[rows])
        miss = np.flatnonzero(~anyl)
        if len(miss):
            out[miss, col] = empty_value(tree, pts[miss])
    return out


# --------------------------------------------------------------------------
# Rendering (render.py:43-448)

@dataclass
class RenderParams:
    """RenderConfig defaults (render.py:91-105)."""
    delta: float = 0.0003
    max_iters: int = 200
    far_plane: float = 5.0
    lod: float | None = None
    normal_eps: float | None = None
    skip_eps: float = 1e-5
    osc_factor: float = 6.0
    light_dir: tuple = (-0.45, 0.8, -0.55)
    albedo: tuple = (0.82, 0.84, 0.88)
    ambient: float = 0.12
    background: tuple = (0.09, 0.10, 0.13)
    shadows: bool = False           # extension (configs[4]); not in the reference
    shadow_offset: float | None = None


def camera_rays(position, look_at, up, fov_y_deg, width, height):
    """Camera.rays (render.py:66-88): pixel-centre rays, row 0 at the top."""
    pos = np.asarray(position, dtype=np.float64)
    f = np.asarray(look_at, dtype=np.float64) - pos
    f = f / np.linalg.norm(f)
    r = np.cross(f, np.asarray(up, dtype=np.float64))
    r = r / np.linalg.norm(r)
    u = np.cross(r, f)
    th = math.tan(math.radians(fov_y_deg) / 2.0)
    px = (2.0 * (np.arange(width) + 0.5) / width - 1.0) * th * (width / height)
    py = (1.0 - 2.0 * (np.arange(height) + 0.5) / height) * th
    d = (f[None, None, :] + px[None, :, None] * r[None, None, :]
         + py[:, None, None] * u[None, None, :]).reshape(-1, 3)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.broadcast_to(pos, d.shape).copy(), d


def query(tree, Z, decoders, pts, lod: float, counts: Counts | None = None) -> np.ndarray:
    """query_field (render.py:155-171): decode only inside trace-level voxels."""
    lvl = min(int(math.ceil(max(lod, 1.0))), tree.max_level)
    inside = locate(tree, pts, lvl) >= 0
    out = np.empty(len(pts))
    rows = np.flatnonzero(inside)
    if len(rows):
        out[rows] = blend(tree, Z, decoders, pts[rows], lod, counts)
    miss = np.flatnonzero(~inside)
    if len(miss):
        out[miss] = empty_value(tree, pts[miss])
        if counts is not None:
            counts.empty_fallbacks += len(miss)
    return out


def march(tree, Z, decoders, origins, dirs, final: PairList, lod: float,
          cfg: RenderParams, counts: Counts | None = None, sdf_fn=None):
    """sphere_trace (render.py:174-274) with per-ray advance semantics.

    `sdf_fn(pts) -> d` replaces the field lookup (the reference's tests
    monkeypatch render.query_field the same way, test_render.py:159-219).
    Returns (hit, t_hit, iters, evals).
    """
    n = len(origins)
    hit = np.zeros(n, dtype=bool)
    t_hit = np.full(n, np.nan)
    iters = np.zeros(n, dtype=np.int32)
    evals = np.zeros(n, dtype=np.int64)
    if len(final) == 0:
        return hit, t_hit, iters, evals
    seg_lo, seg_hi = segments(final, n)
    blo, bhi = voxel_boxes(tree, final.level, final.voxels)
    te, tx = final.t_enter, final.t_exit
    cur = seg_lo.copy()
    t = np.zeros(n)
    prev = np.full(n, np.nan)
    alive = cur < seg_hi
    passes = 1 if float(lod) == int(lod) or lod <= 1.0 else 2
    osc = cfg.osc_factor * cfg.delta
    while True:
        # per-ray advance to the next query point (render.py:202-238)
        pending = np.flatnonzero(alive)
        while len(pending):
            gone = cur[pending] >= seg_hi[pending]
            gone |= t[pending] > cfg.far_plane
            alive[pending[gone]] = False
            pending = pending[~gone]
            if not len(pending):
                break
            c = cur[pending]
            passed = t[pending] >= tx[c]
            cur[pending[passed]] += 1
            prev[pending[passed]] = np.nan
            rest = pending[~passed]
            c = cur[rest]
            early = t[rest] < te[c]
            e_rows = rest[early]
            t_in = te[cur[e_rows]] + cfg.skip_eps
            sliver = t_in >= tx[cur[e_rows]]
            cur[e_rows[sliver]] += 1
            t[e_rows[~sliver]] = t_in[~sliver]
            pending = np.concatenate([pending[passed], e_rows[sliver]])
            pending.sort()
        a = np.flatnonzero(alive)
        if not len(a):
            break
        c = cur[a]
        x = origins[a] + t[a, None] * dirs[a]
        x = np.clip(x, blo[c], bhi[c] - (bhi[c] - blo[c]) * 1e-9)   # clamp_into, octree.py:293-300
        d = sdf_fn(x) if sdf_fn is not None else query(tree, Z, decoders, x, lod, counts)
        evals[a] += passes
        iters[a] += 1
        p = prev[a]
        is_hit = d < cfg.delta
        with np.errstate(invalid="ignore"):
            stalled = ~is_hit & (d >= p) & (np.abs(d - p) < osc)
        h = a[is_hit]
        hit[h] = True
        t_hit[h] = t[h] + d[is_hit]
        alive[h] = False
        alive[a[stalled]] = False
        go = ~is_hit & ~stalled
        g = a[go]
        capped = iters[g] >= cfg.max_iters
        alive[g[capped]] = False
        g2 = g[~capped]
        dg = d[go][~capped]
        prev[g2] = dg
        t[g2] += dg
    return hit, t_hit, iters, evals


def normals(tree, Z, decoders, pts, eps: float, lod: float, counts: Counts | None = None):
    """normals (render.py:277-300): 6 clipped central-difference probes."""
    p = np.atleast_2d(np.asarray(pts, dtype=np.float64))
    k = len(p)
    if k == 0:
        return np.zeros((0, 3)), np.zeros(0, dtype=bool)
    step = eps * np.eye(3)
    probes = np.concatenate([p[:, None, :] + step[None], p[:, None, :] - step[None]], axis=1).reshape(-1, 3)
    np.clip(probes, DMIN, DMAX, out=probes)
    v = query(tree, Z, decoders, probes, lod, counts).reshape(k, 2, 3)
    g = (v[:, 0, :] - v[:, 1, :]) / (2.0 * eps)
    nrm = np.linalg.norm(g, axis=1)
    ok = np.isfinite(nrm) & (nrm > 1e-12)
    out = np.zeros((k, 3))
    out[ok] = g[ok] / nrm[ok, None]
    return out, ok


def shade(hit, nrm, cfg: RenderParams, shadowed=None) -> np.ndarray:
    """shade (render.py:303-314): Lambert, 8-bit; shadowed pixels keep only
    the ambient term (shadow extension)."""
    light = np.asarray(cfg.light_dir, dtype=np.float64)
    light = light / np.linalg.norm(light)
    lam = np.clip(nrm @ light, 0.0, 1.0)
    if shadowed is not None:
        lam = np.where(shadowed, 0.0, lam)
    rgb = np.where(hit[..., None],
                   np.asarray(cfg.albedo) * (cfg.ambient + (1.0 - cfg.ambient) * lam[..., None]),
                   np.asarray(cfg.background))
    return (np.clip(rgb, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)


@dataclass
class OracleFrame:
    hit: np.ndarray
    t: np.ndarray
    points: np.ndarray
    normal: np.ndarray
    normal_ok: np.ndarray
    iterations: np.ndarray
    evals: np.ndarray
    color: np.ndarray
    total_evals: int
    visible: int
    lod: float
    shadowed: np.ndarray | None = None


def render(tree, Z, decoders, camera: dict, cfg: RenderParams, shard: int = 8192,
           ray_slice=None, workers: int = 1) -> OracleFrame:
    """render (render.py:342-448). `camera` holds position, look_at, up,
    fov_y_deg, width, height. `ray_slice` (a slice or an index array)
    restricts the frame to a subset of pixels (bounded CPU samples for the
    bench); `workers` shards the march over threads like the reference
    (render.py:389-414)."""
    L = tree.max_level
    lod = float(cfg.lod) if cfg.lod is not None else float(L)
    if lod > L:
        raise OracleError(f"lod {lod} above max level {L}")
    lod = max(lod, 1.0)
    level = min(int(math.ceil(lod)), L)
    eps = cfg.normal_eps if cfg.normal_eps is not None else 0.5 * tree.edge(L)
    o, d = camera_rays(camera["position"], camera["look_at"], camera["up"],
                       camera["fov_y_deg"], camera["width"], camera["height"])
    if ray_slice is not None:
        o, d = o[ray_slice], d[ray_slice]
    n = len(o)
    fin = traverse(tree, o, d, level)[-1]
    lo_seg, hi_seg = segments(fin, n)
    hit = np.zeros(n, dtype=bool)
    t_hit = np.full(n, np.nan)
    iters = np.zeros(n, dtype=np.int32)
    evals = np.zeros(n, dtype=np.int64)
    shards = [slice(s, min(s + shard, n)) for s in range(0, n, shard)]

    def do_shard(sl):
        c = Counts()
        a, b = lo_seg[sl.start], hi_seg[sl.stop - 1]
        sub = PairList(fin.level, fin.rays[a:b] - sl.start, fin.voxels[a:b], fin.t_enter[a:b], fin.t_exit[a:b])
        hit[sl], t_hit[sl], iters[sl], evals[sl] = march(tree, Z, decoders, o[sl], d[sl], sub, lod, cfg, c)
        return c

    def run(fn, items):
        if workers > 1 and len(items) > 1:
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(workers) as pool:
                return list(pool.map(fn, items))
        return [fn(i) for i in items]

    counts = run(do_shard, shards)
    pts = np.zeros((n, 3))
    pts[hit] = o[hit] + t_hit[hit, None] * d[hit]
    nrm = np.zeros((n, 3))
    ok = np.zeros(n, dtype=bool)
    hot = np.flatnonzero(hit)

    def do_normals(sl):
        c = Counts()
        rows = hot[sl]
        nrm[rows], ok[rows] = normals(tree, Z, decoders, pts[rows], eps, lod, c)
        return c

    counts += run(do_normals, [slice(s, min(s + shard, len(hot))) for s in range(0, len(hot), shard)])
    shadowed = None
    if cfg.shadows and len(hot):
        # secondary rays: the reference's composition for arbitrary rays
        # (metrics.trace_field_rays, metrics.py:135-142) from p + off * n
        off = cfg.shadow_offset if cfg.shadow_offset is not None else 2.0 * eps
        light = np.asarray(cfg.light_dir, dtype=np.float64)
        light = light / np.linalg.norm(light)
        so = pts[hot] + off * nrm[hot]
        sd = np.broadcast_to(light, so.shape).copy()
        sfin = traverse(tree, so, sd, level)[-1]
        c = Counts()
        shit, _, _, _ = march(tree, Z, decoders, so, sd, sfin, lod, cfg, c)
        counts.append(c)
        shadowed = np.zeros(n, dtype=bool)
        shadowed[hot] = shit
    total = sum(c.decoder_evals for c in counts)
    if sum(c.evals_missing_level for c in counts):
        raise OracleError("decoder ran outside the queried level's voxels")
    if ray_slice is None:
        h, w = camera["height"], camera["width"]
        shp = (h, w)
    else:
        shp = (n,)
    color = shade(hit.reshape(shp), nrm.reshape(shp + (3,)), cfg,
                  None if shadowed is None else shadowed.reshape(shp))
    return OracleFrame(hit.reshape(shp), t_hit.reshape(shp), pts.reshape(shp + (3,)),
                       nrm.reshape(shp + (3,)), ok.reshape(shp), iters.reshape(shp),
                       evals.reshape(shp), color, int(total), int(hit.sum()), lod,
                       None if shadowed is None else shadowed.reshape(shp))


# --------------------------------------------------------------------------
# Synthetic shapes used by the parity cases (host ground truth; the
# reference's analytic primitives geometry.py:141-149 plus the torus knot of
# SURVEY.md Appendix A, which has no reference primitive).

def sdf_sphere(radius: float):
    def f(p):
        return np.linalg.norm(np.atleast_2d(p), axis=-1) - radius
    return f


def sdf_torus(major: float, minor: float):
    def f(p):
        p = np.atleast_2d(p)
        ring = np.hypot(p[:, 0], p[:, 2]) - major
        return np.hypot(ring, p[:, 1]) - minor
    return f


def knot_polyline(segments: int = 1024, p: int = 2, q: int = 3, R: float = 0.5,
                  r: float = 0.2, scale: float = 1.2) -> np.ndarray:
    t = np.arange(segments) * (2.0 * np.pi / segments)
    rho = R + r * np.cos(q * t)
    return np.stack([rho * np.cos(p * t), r * np.sin(q * t), rho * np.sin(p * t)], axis=1) * scale


def sdf_polyline_tube(verts: np.ndarray, tube: float, chunk: int = 4096):
    """Distance to a closed polyline minus the tube radius (1-Lipschitz)."""
    a = np.asarray(verts, dtype=np.float64)
    b = np.roll(a, -1, axis=0)
    ab = b - a
    ab2 = np.einsum("ij,ij->i", ab, ab)

    def f(pts):
        pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
        out = np.empty(len(pts))
        for s in range(0, len(pts), chunk):
            p = pts[s:s + chunk]
            ap = p[:, None, :] - a[None, :, :]
            h = np.clip(np.einsum("kij,ij->ki", ap, ab) / ab2[None, :], 0.0, 1.0)
            diff = ap - h[:, :, None] * ab[None, :, :]
            out[s:s + chunk] = np.sqrt(np.einsum("kij,kij->ki", diff, diff).min(axis=1)) - tube
        return out
    return f


def plant_field(tree: OracleOctree, Z: np.ndarray, decoders: list, sdf) -> tuple:
    """The deterministic "planted" field of SURVEY.md Appendix A: decoder L
    reads feature channel L-1, which holds the true SDF at level-L corners."""
    Z = Z.copy()
    decs = [OracleDecoder(d.W1.copy(), d.b1.copy(), d.W2.copy(), d.b2.copy()) for d in decoders]
    for L in range(1, tree.max_level + 1):
        res = tree.res(L)
        ijk = morton_decode(tree.codes[L])
        pos = (DMIN + (ijk[:, None, :] + CORNER_OFS[None]) * (SPAN / res)).reshape(-1, 3)
        ids = tree.corners[L].ravel()
        Z[ids, L - 1] = np.asarray(sdf(pos)).astype(np.float32)
        d = decs[L - 1]
        d.W1[0:2, :] = 0.0
        d.b1[0:2] = 0.0
        d.W1[0, 3 + L - 1] = 1.0
        d.W1[1, 3 + L - 1] = -1.0
        d.W2[:] = 0.0
        d.W2[0, 0] = 1.0
        d.W2[0, 1] = -1.0
        d.b2[:] = 0.0
    return Z, decs
