"""CPU oracle for the NGLOD training step -- TEST INFRASTRUCTURE ONLY.

NumPy restatement of the reference's training path:
the field backward pass (octfield/field.py:286-409), the loss / Adam /
schedule / epoch loop (octfield/trainer.py:1-296) and the epoch sampler it
draws from (octfield/sampling.py:1-196). Only `tests/` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it; the
product package never does.

Pinned by `tests/golden/make_golden.py` (train.npz: the real reference's
gradients, hand loss, Adam steps, sample sets and short training runs) and,
where /root/reference is importable, live in `tests/test_oracle.py`.

Arithmetic is float64 with the reference's operation order; the merge of
per-chunk partial gradients follows trainer.py:254-280 (fixed 128-row chunks
summed in chunk order), so results are bit-identical to the reference on
the same machine's BLAS.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .nglod_oracle import OracleDecoder, OracleError, empty_value, interp

ADAM_BETA1 = 0.9     # trainer.py:29
ADAM_BETA2 = 0.999   # trainer.py:30
ADAM_EPS = 1e-8      # trainer.py:31
CHUNK = 128          # trainer.py:33

SCHEME_SURFACE, SCHEME_NEAR, SCHEME_UNIFORM = 0, 1, 2  # sampling.py:22-24
NEAR_SIGMA = 0.01        # sampling.py:27
SURFACE_HIT_TOL = 1e-3   # sampling.py:28
HIT_RATE_FLOOR = 1e-4    # sampling.py:29


class Diverged(OracleError):
    """TrainingDiverged (errors.py)."""


# --------------------------------------------------------------------------
# backward (field.py:286-409)

def f64_decoder(d) -> OracleDecoder:
    return OracleDecoder(*(np.array(a, dtype=np.float64) for a in (d.W1, d.b1, d.W2, d.b2)))


@dataclass
class Grads:
    """FieldGradients (field.py:294-318): dZ plus one optional slot per decoder."""

    dZ: np.ndarray
    dec: list  # None or [W1, b1, W2, b2]

    @classmethod
    def zeros(cls, Z, n_dec: int) -> "Grads":
        return cls(np.zeros(np.shape(Z)), [None] * n_dec)

    def slot(self, L: int, d) -> list:
        if self.dec[L - 1] is None:
            self.dec[L - 1] = [np.zeros(np.shape(a)) for a in (d.W1, d.b1, d.W2, d.b2)]
        return self.dec[L - 1]


@dataclass
class Cache:
    """ForwardCache (field.py:321-334)."""

    Z: np.ndarray
    decoder: OracleDecoder
    L: int
    pts: np.ndarray
    recs: list
    rows: np.ndarray
    inp: np.ndarray
    pre: np.ndarray
    out: np.ndarray


def forward(tree, Z, decoders, x, L: int):
    """forward (field.py:337-357): predict plus the backward cache."""
    pts = np.atleast_2d(np.asarray(x, dtype=np.float64))
    if not 1 <= L <= len(decoders):
        raise OracleError(f"level {L} outside 1..{len(decoders)}")
    recs = [interp(tree, Z, pts, lv) for lv in range(1, L + 1)]
    z = np.zeros((len(pts), Z.shape[1]))
    anyl = np.zeros(len(pts), dtype=bool)
    for r in recs:
        z += r.psi
        anyl |= r.mask
    rows = np.flatnonzero(anyl)
    d = decoders[L - 1]
    inp = np.concatenate([pts[rows], z[rows]], axis=1)
    pre = inp @ d.W1.T.astype(np.float64) + d.b1.astype(np.float64)
    out = np.empty(len(pts))
    out[rows] = (np.maximum(pre, 0.0) @ d.W2.T.astype(np.float64) + d.b2.astype(np.float64))[:, 0]
    miss = np.flatnonzero(~anyl)
    if len(miss):
        out[miss] = empty_value(tree, pts[miss])
    return out, Cache(Z, d, L, pts, recs, rows, inp, pre, out)


def scatter_add_rows(dst, idx, rows) -> None:
    """field.py:397-409: dst[idx] += rows, duplicates summed in stable order."""
    if len(idx) == 0:
        return
    order = np.argsort(idx, kind="stable")
    si = idx[order]
    sr = rows[order]
    starts = np.concatenate([[0], np.flatnonzero(np.diff(si)) + 1])
    dst[si[starts]] += np.add.reduceat(sr, starts, axis=0)


def backward(cache: Cache, upstream, grads: Grads | None = None, n_dec: int | None = None) -> Grads:
    """backward (field.py:360-394): partials of sum(upstream * out)."""
    if grads is None:
        grads = Grads.zeros(cache.Z, n_dec if n_dec is not None else cache.L)
    up = np.atleast_1d(np.asarray(upstream, dtype=np.float64))
    if up.shape != (len(cache.pts),):
        raise OracleError("upstream shape does not match the forward batch")
    rows = cache.rows
    if len(rows) == 0:
        return grads
    d = cache.decoder
    dout = up[rows]
    hidden = np.maximum(cache.pre, 0.0)
    g = grads.slot(cache.L, d)
    g[2] += dout[None, :] @ hidden
    g[3] += dout.sum(keepdims=True)
    dpre = np.where(cache.pre > 0.0, dout[:, None] * d.W2.astype(np.float64), 0.0)
    g[0] += dpre.T @ cache.inp
    g[1] += dpre.sum(axis=0)
    dz = (dpre @ d.W1.astype(np.float64))[:, 3:]
    dz_full = np.zeros((len(cache.pts), dz.shape[1]))
    dz_full[rows] = dz
    for rec in cache.recs:
        r = np.flatnonzero(rec.mask)
        if len(r) == 0:
            continue
        contrib = rec.w[:, :, None] * dz_full[r][:, None, :]
        scatter_add_rows(grads.dZ, rec.ids.ravel(), contrib.reshape(-1, dz.shape[1]))
    return grads


# --------------------------------------------------------------------------
# loss, Adam, schedules (trainer.py:62-162)

def loss_batch(tree, Z, decoders, pts, dist, active, grads: Grads | None = None, denom: int | None = None,
               want_grads: bool = True):
    """loss_batch (trainer.py:106-144): (loss, grads, level_sums)."""
    active = sorted(set(int(v) for v in active))
    if not active:
        raise OracleError("active level set is empty")
    if active[0] < 1 or active[-1] > len(decoders):
        raise OracleError(f"active levels {active} outside 1..{len(decoders)}")
    n = len(pts) if denom is None else denom
    sums = np.zeros(len(decoders))
    if want_grads and grads is None:
        grads = Grads.zeros(Z, len(decoders))
    for L in active:
        out, cache = forward(tree, Z, decoders, pts, L)
        mask = cache.recs[L - 1].mask
        resid = np.where(mask, out - dist, 0.0)
        sums[L - 1] = float(resid @ resid)
        if want_grads:
            backward(cache, (2.0 / n) * resid, grads)
    loss = float(sums[np.array(active) - 1].sum() / n)
    return loss, grads, sums


@dataclass
class Adam:
    """AdamState (trainer.py:62-84)."""

    m: dict
    v: dict
    step: int = 0

    @classmethod
    def for_params(cls, params: dict) -> "Adam":
        return cls({k: np.zeros(p.shape) for k, p in params.items()},
                   {k: np.zeros(p.shape) for k, p in params.items()})


def adam_step(params: dict, grads: dict, st: Adam, lr: float) -> None:
    """adam_step (trainer.py:87-103), in place; params without a gradient are untouched."""
    st.step += 1
    c1 = 1.0 - ADAM_BETA1 ** st.step
    c2 = 1.0 - ADAM_BETA2 ** st.step
    for name, g in grads.items():
        if not np.all(np.isfinite(g)):
            raise Diverged(f"non-finite gradient for {name}")
        m = st.m[name]
        v = st.v[name]
        m *= ADAM_BETA1
        m += (1.0 - ADAM_BETA1) * g
        v *= ADAM_BETA2
        v += (1.0 - ADAM_BETA2) * (g * g)
        params[name] -= lr * (m / c1) / (np.sqrt(v / c2) + ADAM_EPS)


def active_levels_for(schedule: str, epoch: int, interval: int, max_level: int) -> list:
    """trainer.py:154-162."""
    if schedule == "progressive":
        k = min(1 + epoch // interval, max_level)
        return list(range(max_level - k + 1, max_level + 1))
    return list(range(1, max_level + 1))


# --------------------------------------------------------------------------
# sampling (sampling.py:46-167), analytic oracles only

DOMAIN_MIN, DOMAIN_MAX = -1.0, 1.0


def sample_uniform(count: int, seed: int) -> np.ndarray:
    """sampling.py:46-49."""
    return np.random.default_rng(seed).uniform(DOMAIN_MIN, DOMAIN_MAX, size=(count, 3))


def _bisect(sdf, o, d, t_lo, t_hi, side, iters: int = 40):
    """_bisect_crossing (sampling.py:142-149)."""
    for _ in range(iters):
        mid = 0.5 * (t_lo + t_hi)
        hi_side = side * sdf(o + mid[:, None] * d) < 0.0
        t_hi = np.where(hi_side, mid, t_hi)
        t_lo = np.where(hi_side, t_lo, mid)
    return 0.5 * (t_lo + t_hi)


def _trace(sdf, o, d, tol, t_max, max_iters: int = 128):
    """_trace_to_surface (sampling.py:109-139)."""
    f0 = sdf(o)
    side = np.where(f0 < 0.0, -1.0, 1.0)
    t = np.zeros(len(o))
    f_prev = side * f0
    t_prev = t.copy()
    alive = np.abs(f0) >= tol
    hit_t = np.full(len(o), np.nan)
    hit_t[~alive] = 0.0
    for _ in range(max_iters):
        if not alive.any():
            break
        idx = np.flatnonzero(alive)
        t[idx] = t[idx] + f_prev[idx]
        over = t[idx] > t_max
        f = side[idx] * sdf(o[idx] + t[idx, None] * d[idx])
        done = (np.abs(f) < tol) & ~over
        hit_t[idx[done]] = t[idx[done]]
        crossed = (f < 0.0) & ~done & ~over
        if crossed.any():
            j = idx[crossed]
            hit_t[j] = _bisect(sdf, o[j], d[j], t_prev[j], t[j], side[j])
        stop = done | crossed | over
        f_prev[idx] = f
        t_prev[idx] = t[idx]
        alive[idx[stop]] = False
    ok = np.isfinite(hit_t)
    return o[ok] + hit_t[ok, None] * d[ok]


def surface_points(sdf, count: int, seed: int, tol: float = SURFACE_HIT_TOL) -> np.ndarray:
    """sample_surface_sdf (sampling.py:68-106) for an analytic sdf callable."""
    if count == 0:
        return np.zeros((0, 3))
    rng = np.random.default_rng(seed)
    hits = []
    got = cast = 0
    t_max = 2.0 * np.sqrt(3.0) * (DOMAIN_MAX - DOMAIN_MIN) / 2.0
    while got < count:
        k = max(4 * (count - got), 4096)
        o = rng.uniform(DOMAIN_MIN, DOMAIN_MAX, size=(k, 3))
        d = rng.standard_normal((k, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        p = _trace(sdf, o, d, tol, t_max)
        cast += k
        if len(p):
            hits.append(p)
            got += len(p)
        if cast >= 100000 and got / cast < HIT_RATE_FLOOR:
            raise OracleError("surface hit rate below floor")
    return np.concatenate(hits)[:count]


def split_counts(total: int):
    """sampling.py:159-164."""
    uni = total // 5
    near = (2 * total) // 5
    return total - near - uni, near, uni


def epoch_set(sdf, total: int, seed: int, sigma: float = NEAR_SIGMA):
    """build_epoch_set (sampling.py:177-196): (points, distances, tags)."""
    ns, nn, nu = split_counts(total)
    s = int(np.random.SeedSequence(seed).generate_state(1)[0])
    surf = surface_points(sdf, ns + nn, s)
    near = np.clip(surf[ns:] + sigma * np.random.default_rng(s + 1).standard_normal(surf[ns:].shape),
                   DOMAIN_MIN, DOMAIN_MAX)
    uni = sample_uniform(nu, s + 2)
    pts = np.concatenate([surf[:ns], near, uni])
    tags = np.concatenate([np.full(ns, SCHEME_SURFACE, np.int8), np.full(nn, SCHEME_NEAR, np.int8),
                           np.full(nu, SCHEME_UNIFORM, np.int8)])
    return pts, sdf(pts), tags


# --------------------------------------------------------------------------
# the epoch loop (trainer.py:165-296)

def _batch_pass(tree, Z, decoders, pts, dist, active):
    """_batch_pass (trainer.py:254-280): 128-row chunks merged in order."""
    n = len(pts)
    total = Grads.zeros(Z, len(decoders))
    loss = 0.0
    sums = np.zeros(len(decoders))
    for s in range(0, n, CHUNK):
        sl = slice(s, min(s + CHUNK, n))
        part_loss, g, part_sums = loss_batch(tree, Z, decoders, pts[sl], dist[sl], active,
                                             Grads.zeros(Z, len(decoders)), denom=n)
        loss += part_loss
        sums += part_sums
        total.dZ += g.dZ
        for i, gd in enumerate(g.dec):
            if gd is None:
                continue
            if total.dec[i] is None:
                total.dec[i] = [a.copy() for a in gd]
            else:
                for a, b in zip(total.dec[i], gd):
                    a += b
    return loss, total, sums


def train(tree, Z, decoders, sdf, epochs: int, points_per_epoch: int = 500_000, batch_size: int = 512,
          lr: float = 0.001, schedule: str = "joint", interval: int = 100, seed: int = 0):
    """train (trainer.py:165-251). Returns (Z64, decoders64, history) where
    history rows are the per-level epoch losses (nan where inactive)."""
    Z = np.array(Z, dtype=np.float64)
    decs = [f64_decoder(d) for d in decoders]
    hist = []
    if epochs == 0:
        return Z, decs, hist
    params = {"Z": Z}
    for i, d in enumerate(decs):
        params[f"decoder{i + 1}.W1"] = d.W1
        params[f"decoder{i + 1}.b1"] = d.b1
        params[f"decoder{i + 1}.W2"] = d.W2
        params[f"decoder{i + 1}.b2"] = d.b2
    st = Adam.for_params(params)
    upd = schedule != "frozen_decoder"
    Lm = len(decs)
    for ep in range(epochs):
        seeds = np.random.SeedSequence([seed, ep]).generate_state(2)
        pts, dist, _ = epoch_set(sdf, points_per_epoch, int(seeds[0]))
        perm = np.random.default_rng(int(seeds[1])).permutation(len(pts))
        pts, dist = pts[perm], dist[perm]
        active = active_levels_for(schedule, ep, interval, Lm)
        ep_sums = np.zeros(Lm)
        for s in range(0, len(pts), batch_size):
            e = min(s + batch_size, len(pts))
            loss, g, sums = _batch_pass(tree, Z, decs, pts[s:e], dist[s:e], active)
            ep_sums += sums
            if not np.isfinite(loss):
                raise Diverged(f"epoch {ep}, batch at {s}: loss {loss}")
            gd = {"Z": g.dZ}
            if upd:
                for i, slot in enumerate(g.dec):
                    if slot is None:
                        continue
                    for nm, a in zip(("W1", "b1", "W2", "b2"), slot):
                        gd[f"decoder{i + 1}.{nm}"] = a
            adam_step(params, gd, st, lr)
        losses = np.full(Lm, np.nan)
        idx = np.array(active) - 1
        losses[idx] = ep_sums[idx] / len(pts)
        hist.append(losses)
    return Z, decs, hist
