"""The neural distance field, evaluated on the GPU.

Drop-in for octfield.field (field.py:1-413, forward path). A flat feature
volume Z holds one m-vector per unique voxel corner; a query at level L
trilinearly interpolates the containing voxel's corners at every feature
level 1..L, sums them and decodes [x, z] with level L's MLP. Parameters are
fp32 (as the reference stores them); the device computes the gather and the
MLP in fp32 and the geometry (binning, weights' local coordinates, empty-
space values, blends) in fp64, which keeps SDF values within 1e-4 of the
reference's all-fp64 path.

Device layout: Z is padded to 32 channels (128-byte rows, one coalesced
line per corner); decoders are packed per level as W1b[h][36] = (x weights,
feature weights, b1), W2[h], b2 (include/nglod_b200.h, ng_field).
"""

from __future__ import annotations

import ctypes
import threading
import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream_ptr
from .errors import OctfieldError, StructuralError
from .octree import DOMAIN_MAX, DOMAIN_MIN, SparseVoxelOctree

FEATURE_DIM = 32
HIDDEN_DIM = 128
FEATURE_INIT_SIGMA = 0.01


@dataclass
class Decoder:
    """Single-hidden-layer MLP weights for one detail level (field.py:30-48)."""

    W1: np.ndarray  # (h, 3 + m)
    b1: np.ndarray  # (h,)
    W2: np.ndarray  # (1, h)
    b2: np.ndarray  # (1,)

    def param_count(self) -> int:
        return self.W1.size + self.b1.size + self.W2.size + self.b2.size

    def astype(self, dtype) -> "Decoder":
        return Decoder(self.W1.astype(dtype), self.b1.astype(dtype), self.W2.astype(dtype), self.b2.astype(dtype))


def init_features(svo: SparseVoxelOctree, m: int = FEATURE_DIM, seed: int = 0) -> np.ndarray:
    """Gaussian features, one row per unique corner (field.py:51-56)."""
    rng = np.random.default_rng(seed)
    return (FEATURE_INIT_SIGMA * rng.standard_normal((svo.corner_count, m))).astype(np.float32)


def init_decoders(max_level: int, m: int = FEATURE_DIM, h: int = HIDDEN_DIM, seed: int = 0) -> list:
    """Uniform fan-in init, one decoder per level (field.py:59-76)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(max_level):
        k1 = 1.0 / np.sqrt(3 + m)
        k2 = 1.0 / np.sqrt(h)
        out.append(Decoder(
            rng.uniform(-k1, k1, size=(h, 3 + m)).astype(np.float32),
            rng.uniform(-k1, k1, size=h).astype(np.float32),
            rng.uniform(-k2, k2, size=(1, h)).astype(np.float32),
            rng.uniform(-k2, k2, size=1).astype(np.float32),
        ))
    return out


class EvalCounter:
    """Tallies decoder work (field.py:79-90)."""

    def __init__(self):
        self.decoder_evals = 0
        self.evals_missing_level = 0
        self.empty_fallbacks = 0

    def reset(self):
        self.decoder_evals = 0
        self.evals_missing_level = 0
        self.empty_fallbacks = 0

    def add(self, c) -> None:
        self.decoder_evals += int(c[0])
        self.evals_missing_level += int(c[1])
        self.empty_fallbacks += int(c[2])


def decoder_stride(h: int) -> int:
    return h * _lib.W1_STRIDE + ((h + 1 + 3) // 4) * 4


def pack_decoders(decoders: list, m: int) -> np.ndarray:
    """Pack per-level decoders into the device layout (ng_field)."""
    if m > _lib.FEAT_PAD:
        raise StructuralError(f"feature dim {m} above the device limit {_lib.FEAT_PAD}")
    h = decoders[0].W1.shape[0]
    stride = decoder_stride(h)
    buf = np.zeros((len(decoders), stride), dtype=np.float32)
    for i, d in enumerate(decoders):
        W1 = np.asarray(d.W1, dtype=np.float32)
        if W1.shape != (h, 3 + m):
            raise StructuralError("decoders must share (h, 3 + m) shapes")
        blk = buf[i, :h * _lib.W1_STRIDE].reshape(h, _lib.W1_STRIDE)
        blk[:, 0:3 + m] = W1
        blk[:, 35] = np.asarray(d.b1, dtype=np.float32).ravel()
        buf[i, h * _lib.W1_STRIDE:h * _lib.W1_STRIDE + h] = np.asarray(d.W2, dtype=np.float32).ravel()
        buf[i, h * _lib.W1_STRIDE + h] = np.float32(np.asarray(d.b2).ravel()[0])
    return buf


def pack_decoders64(decoders: list, m: int, h: int) -> np.ndarray:
    """fp64 decoder blocks, W1b[h][36] | W2[h] | b2 (the training layout)."""
    stride = decoder_stride(h)
    buf = np.zeros((len(decoders), stride), dtype=np.float64)
    for i, d in enumerate(decoders):
        W1 = np.asarray(d.W1, dtype=np.float64)
        if W1.shape != (h, 3 + m):
            raise StructuralError("decoders must share (h, 3 + m) shapes")
        blk = buf[i, :h * _lib.W1_STRIDE].reshape(h, _lib.W1_STRIDE)
        blk[:, :3 + m] = W1
        blk[:, _lib.W1_STRIDE - 1] = np.asarray(d.b1, dtype=np.float64).ravel()
        buf[i, h * _lib.W1_STRIDE:h * (_lib.W1_STRIDE + 1)] = np.asarray(d.W2, dtype=np.float64).ravel()
        buf[i, h * (_lib.W1_STRIDE + 1)] = float(np.asarray(d.b2, dtype=np.float64).ravel()[0])
    return buf


class DeviceField:
    """Device copies of Z (padded to 32 channels) and the packed decoders."""

    def __init__(self, Z, decoders: list):
        dev = _lib.device()
        if isinstance(Z, torch.Tensor):
            m = Z.shape[1]
            z = Z.to(device=dev, dtype=torch.float32)
        else:
            Zn = np.asarray(Z)
            m = Zn.shape[1]
            z = torch.from_numpy(np.ascontiguousarray(Zn, dtype=np.float32)).to(dev)
        if m > _lib.FEAT_PAD:
            raise StructuralError(f"feature dim {m} above the device limit {_lib.FEAT_PAD}")
        if m < _lib.FEAT_PAD:
            zp = torch.zeros((z.shape[0], _lib.FEAT_PAD), dtype=torch.float32, device=dev)
            zp[:, :m] = z
            z = zp
        self.Z = z.contiguous()
        self.m = m
        self.h = decoders[0].W1.shape[0]
        self.n_decoders = len(decoders)
        self.dec = torch.from_numpy(pack_decoders(decoders, m)).to(dev)
        s = _lib.NgField()
        s.Z = ptr(self.Z)
        s.decoders = ptr(self.dec)
        s.m, s.h, s.n_decoders = m, self.h, self.n_decoders
        s.dec_stride = decoder_stride(self.h)
        s.corner_count = self.Z.shape[0]
        self.struct = s
        self.presum = None
        self._presum_key = None
        self._src = (Z, decoders)
        self._exact = None
        self._tables = {}   # (level, output mask) -> presummed tables, owner ids
        self._lock = threading.Lock()

    def ref(self):
        return ctypes.byref(self.struct)

    def exact(self):
        """fp64 copies of the parameters as given, for the reference-semantics
        API (csrc/exact.cu): Z (C, m) and the decoders in the training
        layout. Made on first use."""
        if self._exact is None:
            Z, decoders = self._src
            dev = self.Z.device
            if isinstance(Z, torch.Tensor):
                z64 = Z.to(device=dev, dtype=torch.float64).contiguous()
            else:
                z64 = torch.from_numpy(np.ascontiguousarray(np.asarray(Z), dtype=np.float64)).to(dev)
            self._exact = (z64, torch.from_numpy(pack_decoders64(decoders, self.m, self.h)).to(dev))
        return self._exact

    def build_presum(self, svo, level: int, out_mask: int):
        """Build the presummed feature tables S_L on the level's corner ids
        that the sphere tracer and the normal probes read instead of
        gathering every level (csrc/presum.cu). Returns (tables, owner)."""
        dev = self.Z.device
        offset = int(svo.corner_offsets[level])
        end = int(svo.corner_offsets[level + 1]) if level < svo.max_level else int(svo.corner_count)
        n = end - offset
        n_out = bin(out_mask).count("1")
        S = torch.empty((n_out, max(n, 1), _lib.FEAT_PAD), dtype=torch.float32, device=dev)
        owner = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        call("ng_field_presum", svo.device.ref(), ptr(self.Z), int(level), int(out_mask), offset, n, ptr(S),
             ptr(owner), stream_ptr())
        return S, owner

    def presum_struct(self, svo, level: int, out_mask: int) -> _lib.NgField:
        """A copy of the field struct carrying the presummed tables of
        (level, output levels), built on first use and kept with the field.
        Each frame launches with its own copy, so frames of different LODs
        may run concurrently on one field."""
        key = (int(level), int(out_mask))
        with self._lock:
            t = self._tables.get(key)
            if t is None:
                t = self._tables[key] = self.build_presum(svo, *key)
            self.presum, self._presum_key = t[0], key
        s = _lib.NgField.from_buffer_copy(self.struct)
        offset = int(svo.corner_offsets[level])
        s.presum = ptr(t[0])
        s.presum_offset = offset
        s.presum_corners = (int(svo.corner_offsets[level + 1]) if level < svo.max_level else int(svo.corner_count)) \
            - offset
        s.presum_level = key[0]
        s.presum_mask = key[1]
        return s


def _as_points(x):
    pts = np.asarray(x, dtype=np.float64)
    single = pts.ndim == 1
    return np.atleast_2d(pts), single


def _check_level(L, max_level):
    if not 1 <= L <= max_level:
        raise StructuralError(f"level {L} outside 1..{max_level}")


class _Counters:
    def __init__(self):
        self.t = torch.zeros(4, dtype=torch.int64, device=_lib.device())

    def ptr(self):
        return ptr(self.t)

    def host(self):
        return self.t.cpu().numpy()


def _run_query(svo, dfield: DeviceField, pts_dev: torch.Tensor, out_levels=0, inside_level=-1,
               blend_base=0, blend_alpha=0.0, ncols=1, counter: EvalCounter | None = None,
               out: torch.Tensor | None = None) -> torch.Tensor:
    n = pts_dev.shape[0]
    if out is None:
        out = torch.empty((n, ncols), dtype=torch.float64, device=pts_dev.device)
    elif (out.dtype != torch.float64 or tuple(out.shape) != (n, ncols) or not out.is_contiguous()
          or out.device != pts_dev.device):
        raise StructuralError(f"out must be a contiguous float64 ({n}, {ncols}) tensor on {pts_dev.device}")
    args = _lib.NgQueryArgs(out_levels, inside_level, blend_base, 0, blend_alpha)
    cnt = _Counters()
    call("ng_query", svo.device.ref(), dfield.ref(), ctypes.byref(args), ptr(pts_dev), n, ptr(out), cnt.ptr(),
         stream_ptr())
    c = cnt.host()
    if c[3]:
        raise OctfieldError("non-finite decoder input")
    if counter is not None:
        counter.add(c)
    return out


def _run_exact(svo, dfield: DeviceField, pts_dev: torch.Tensor, out_levels=0, inside_level=-1, blend_base=0,
               blend_alpha=0.0, ncols=1, counter: EvalCounter | None = None) -> torch.Tensor:
    """predict / blend / query_field with the reference's fp64 semantics
    (csrc/exact.cu, ng_query64)."""
    n = pts_dev.shape[0]
    out = torch.empty((n, ncols), dtype=torch.float64, device=pts_dev.device)
    z64, d64 = dfield.exact()
    args = _lib.NgQueryArgs(out_levels, inside_level, blend_base, 0, blend_alpha)
    cnt = _Counters()
    call("ng_query64", svo.device.ref(), ptr(z64), dfield.m, ptr(d64), dfield.h, dfield.n_decoders,
         decoder_stride(dfield.h), ctypes.byref(args), ptr(pts_dev), n, ptr(out), cnt.ptr(), stream_ptr())
    c = cnt.host()
    if c[3]:
        raise OctfieldError("non-finite decoder input")
    if counter is not None:
        counter.add(c)
    return out


def _dev_points(pts: np.ndarray) -> torch.Tensor:
    if len(pts) and (np.any(pts < DOMAIN_MIN) or np.any(pts > DOMAIN_MAX)):
        raise StructuralError("point outside the domain box")
    return torch.from_numpy(np.ascontiguousarray(pts)).to(_lib.device())


# ---------------------------------------------------------------- interpolation

def trilinear_weights(u: np.ndarray) -> np.ndarray:
    """(k, 8) corner weights from local coordinates (field.py:122-135);
    corner j at offset (j & 1, j >> 1 & 1, j >> 2 & 1). Host helper."""
    u = np.asarray(u, dtype=np.float64)
    cx = np.stack([1.0 - u[:, 0], u[:, 0]], axis=1)
    cy = np.stack([1.0 - u[:, 1], u[:, 1]], axis=1)
    cz = np.stack([1.0 - u[:, 2], u[:, 2]], axis=1)
    j = np.arange(8)
    return cx[:, j & 1] * cy[:, (j >> 1) & 1] * cz[:, (j >> 2) & 1]


def _interp(svo, Z, pts, lo, hi, dfield=None):
    """Per-level interpolation summed over levels lo..hi, in fp64 from the
    parameters as given (ng_interp64)."""
    if dfield is not None:
        z64 = dfield.exact()[0]
    else:
        z64 = torch.from_numpy(np.ascontiguousarray(np.asarray(Z), dtype=np.float64)).to(_lib.device())
    m = int(z64.shape[1])
    if m > _lib.FEAT_PAD:
        raise StructuralError(f"feature dim {m} above the device limit {_lib.FEAT_PAD}")
    n = len(pts)
    z = torch.zeros((n, m), dtype=torch.float64, device=_lib.device())
    mask = torch.zeros((n, hi - lo + 1), dtype=torch.uint8, device=_lib.device())
    if n:
        d = _dev_points(pts)
        call("ng_interp64", svo.device.ref(), ptr(z64), m, ptr(d), n, lo, hi, ptr(z), ptr(mask), stream_ptr())
    return z.cpu().numpy(), mask.cpu().numpy().astype(bool)


def trilinear(svo, Z, x, level: int):
    """Interpolated features at one level (field.py:138-146): (values, mask)."""
    pts, _ = _as_points(x)
    if not 1 <= level <= svo.max_level:
        raise StructuralError(f"level {level} outside 1..{svo.max_level}")
    z, mask = _interp(svo, Z, pts, level, level)
    return z, mask[:, 0]


def sum_features(svo, Z, x, L: int):
    """z(x) = sum of levels 1..L and the (n, L) presence mask (field.py:154-169)."""
    if L < 1:
        raise StructuralError("L must be >= 1")
    pts, _ = _as_points(x)
    return _interp(svo, Z, pts, 1, L)


def decode(decoder: Decoder, x, z):
    """d = W2 relu(W1 [x, z] + b1) + b2 (field.py:172-182), fp64 on device."""
    pts = np.atleast_2d(np.asarray(x, dtype=np.float64))
    z = np.atleast_2d(np.asarray(z, dtype=np.float64))
    inp = np.concatenate([pts, z], axis=1)
    if not np.all(np.isfinite(inp)):
        raise OctfieldError("non-finite decoder input")
    m = z.shape[1]
    h = decoder.W1.shape[0]
    dev = _lib.device()
    if m > _lib.FEAT_PAD:
        raise StructuralError(f"feature dim {m} above the device limit {_lib.FEAT_PAD}")
    blk = torch.from_numpy(pack_decoders64([decoder], m, h)[0]).to(dev)
    n = len(pts)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    if n:
        dx = torch.from_numpy(np.ascontiguousarray(pts)).to(dev)
        dz = torch.from_numpy(np.ascontiguousarray(z)).to(dev)
        call("ng_decode64", ptr(blk), h, m, ptr(dx), ptr(dz), n, ptr(out), ptr(bad), stream_ptr())
    if int(bad.item()):
        raise OctfieldError("non-finite decoder input")
    return out.cpu().numpy()


def empty_space_value(svo: SparseVoxelOctree, x) -> np.ndarray:
    """Distance to the occupied region's AABB + finest half diagonal (field.py:185-191)."""
    pts, _ = _as_points(x)
    n = len(pts)
    out = torch.empty(n, dtype=torch.float64, device=_lib.device())
    if n:
        d = torch.from_numpy(np.ascontiguousarray(pts)).to(_lib.device())
        call("ng_empty_value", svo.device.ref(), ptr(d), n, ptr(out), stream_ptr())
    return out.cpu().numpy()


# ---------------------------------------------------------------- prediction

def predict(svo, Z, decoders, x, L: int, counter: EvalCounter | None = None, _dfield=None):
    """Distance at integer level L (field.py:194-218)."""
    pts, single = _as_points(x)
    _check_level(L, len(decoders))
    df = _dfield if _dfield is not None else DeviceField(Z, decoders)
    out = _run_exact(svo, df, _dev_points(pts), out_levels=1 << (L - 1), counter=counter)[:, 0].cpu().numpy()
    return float(out[0]) if single else out


def blend(svo, Z, decoders, x, L_tilde: float, counter: EvalCounter | None = None, _dfield=None):
    """Continuous-level prediction (field.py:226-239)."""
    if L_tilde > len(decoders):
        raise StructuralError(f"blend level {L_tilde} above max {len(decoders)}")
    L_tilde = max(float(L_tilde), 1.0)
    base = int(np.floor(L_tilde))
    alpha = L_tilde - base
    if alpha == 0.0:
        return predict(svo, Z, decoders, x, base, counter, _dfield)
    pts, single = _as_points(x)
    df = _dfield if _dfield is not None else DeviceField(Z, decoders)
    out = _run_exact(svo, df, _dev_points(pts), blend_base=base, blend_alpha=alpha, counter=counter)
    out = out[:, 0].cpu().numpy()
    return float(out[0]) if single else out


@dataclass
class LevelInterp:
    """Interpolation record for one feature level of a point batch (field.py:93-101)."""

    level: int
    mask: np.ndarray      # (n,)
    ids: np.ndarray       # (k, 8) corner ids of the masked rows
    weights: np.ndarray   # (k, 8) trilinear weights
    psi: np.ndarray       # (n, m), zero where absent


class ForwardCache:
    """What backward needs from a forward pass (field.py:321-334).

    `out` is computed eagerly. The per-level records, decoded rows, decoder
    inputs and pre-activations (`recs`, `rows`, `inp`, `pre`) are exported
    from the device forward pass (ng_train_export) on first access; the
    backward pass itself recomputes them on the device."""

    def __init__(self, svo, Z, decoders, L, pts, out):
        self.svo = svo
        self.Z = Z
        self.decoders = decoders
        self.decoder = decoders[L - 1]
        self.L = L
        self.pts = pts
        self.out = out
        self._export = None

    def _exported(self):
        if self._export is None:
            from .trainer import DeviceTrainState
            st = DeviceTrainState(self.svo, self.Z, self.decoders, moments=False)
            self._export = st.export(self.pts, self.L)
        return self._export

    @property
    def recs(self) -> list:
        return self._exported()["recs"]

    @property
    def rows(self) -> np.ndarray:
        return self._exported()["rows"]

    @property
    def inp(self) -> np.ndarray:
        return self._exported()["inp"]

    @property
    def pre(self) -> np.ndarray:
        return self._exported()["pre"]


def forward(svo, Z, decoders, x, L: int, _dfield=None) -> tuple:
    """predict plus a cache for the matching backward call (field.py:337-357)."""
    pts = np.atleast_2d(np.asarray(x, dtype=np.float64))
    _check_level(L, len(decoders))
    df = _dfield if _dfield is not None else DeviceField(Z, decoders)
    out = _run_exact(svo, df, _dev_points(pts), out_levels=1 << (L - 1))[:, 0].cpu().numpy()
    return out, ForwardCache(svo, Z, decoders, L, pts, out)


@dataclass
class DecoderGrads:
    """field.py:286-291."""

    W1: np.ndarray
    b1: np.ndarray
    W2: np.ndarray
    b2: np.ndarray


@dataclass
class FieldGradients:
    """Accumulated partials for Z and each decoder; decoder slots stay None
    until a backward pass touches that level (field.py:294-318)."""

    dZ: np.ndarray
    decoders: list

    @classmethod
    def zeros(cls, Z, n_decoders: int) -> "FieldGradients":
        return cls(np.zeros(np.shape(Z)), [None] * n_decoders)

    def decoder_slot(self, L: int, decoder: Decoder) -> DecoderGrads:
        g = self.decoders[L - 1]
        if g is None:
            g = DecoderGrads(np.zeros(decoder.W1.shape), np.zeros(decoder.b1.shape), np.zeros(decoder.W2.shape),
                             np.zeros(decoder.b2.shape))
            self.decoders[L - 1] = g
        return g


def backward(cache: ForwardCache, upstream, grads: FieldGradients | None = None) -> FieldGradients:
    """Reverse-mode partials of sum(upstream * out) w.r.t. the level-L decoder
    and every contributing corner feature, accumulated into grads
    (field.py:360-394). Runs on the device in fp64 (csrc/train.cu)."""
    if not isinstance(cache, ForwardCache):
        raise OctfieldError("backward needs the cache returned by forward")
    if grads is None:
        grads = FieldGradients.zeros(cache.Z, cache.svo.max_level)
    up = np.atleast_1d(np.asarray(upstream, dtype=np.float64))
    if up.shape != (len(cache.pts),):
        raise StructuralError("upstream shape does not match the forward batch")
    if len(up) == 0:
        return grads
    from .trainer import DeviceTrainState
    st = DeviceTrainState(cache.svo, cache.Z, cache.decoders, moments=False)
    st.gradients(cache.pts, None, 1 << (cache.L - 1), 1.0, grads, upstream=up)
    return grads


def scatter_add_rows(dst: np.ndarray, idx: np.ndarray, rows: np.ndarray) -> None:
    """dst[idx] += rows with duplicates accumulated (field.py:397-409).
    Host utility kept for API parity; the training step does this
    reduction on the device (k_train_rows)."""
    if len(idx) == 0:
        return
    order = np.argsort(idx, kind="stable")
    idx_s = idx[order]
    starts = np.concatenate([[0], np.flatnonzero(np.diff(idx_s)) + 1])
    dst[idx_s[starts]] += np.add.reduceat(rows[order], starts, axis=0)


def forward_levels_device(svo, dfield: DeviceField, pts: torch.Tensor, levels, counter=None,
                          out: torch.Tensor | None = None) -> torch.Tensor:
    """Batched SDF query on device points: one fp64 column per level in
    `levels` (ascending), each equal to forward(x, L)[0]. All levels share one
    gather pass: z_L is the running prefix sum (the training-forward caller
    trainer.loss_batch, trainer.py:132-142, recomputes 1..L per L). `out`, a
    preallocated (n, len(levels)) float64 device tensor, is written in place
    (a serving loop keeps its output resident instead of allocating per call)."""
    levels = sorted(set(int(v) for v in levels))
    for L in levels:
        _check_level(L, dfield.n_decoders)
    mask = 0
    for L in levels:
        mask |= 1 << (L - 1)
    return _run_query(svo, dfield, pts, out_levels=mask, ncols=len(levels), counter=counter, out=out)


def forward_levels(svo, Z, decoders, x, levels) -> np.ndarray:
    return _host_query(svo, DeviceField(Z, decoders), x, levels)


# ----------------------------------------------------- host arrays in and out

# Points per pipelined chunk of a host query (24 B in, 8 B per level out).
HOST_CHUNK = 1 << 21
_STAGING = threading.local()


class _Staging:
    """Per thread and device: pinned host buffers, device buffers and a copy
    stream for two chunks in flight (reused across calls)."""

    def __init__(self, dev, ncols):
        self.dev, self.ncols = dev, ncols
        self.pin_in = [torch.empty((HOST_CHUNK, 3), dtype=torch.float64, pin_memory=True) for _ in range(2)]
        self.pin_out = [torch.empty((HOST_CHUNK, ncols), dtype=torch.float64, pin_memory=True) for _ in range(2)]
        self.d_in = [torch.empty((HOST_CHUNK, 3), dtype=torch.float64, device=dev) for _ in range(2)]
        self.d_out = [torch.empty((HOST_CHUNK, ncols), dtype=torch.float64, device=dev) for _ in range(2)]
        self.copy = torch.cuda.Stream(dev)


def _staging(dev, ncols) -> _Staging:
    cache = getattr(_STAGING, "d", None)
    if cache is None:
        cache = _STAGING.d = {}
    st = cache.get((dev, ncols))
    if st is None:
        st = cache[(dev, ncols)] = _Staging(dev, ncols)
    return st


def _host_query(svo, dfield: DeviceField, x, levels, counter: EvalCounter | None = None) -> np.ndarray:
    """forward_levels with host arrays: chunks of HOST_CHUNK points go
    numpy -> pinned (torch's multithreaded copy) -> HBM on a copy stream,
    through the query kernel on the caller's stream, and back HBM -> pinned
    -> the result array, two chunks in flight, so the PCIe copies, the
    kernel and the host copies overlap. The domain check
    (StructuralError, octree.py:268-269) runs on the device beside the
    query (points outside are clipped into the domain by the kernels'
    binning, so the query is safe to run first) and is raised before any
    result is returned."""
    levels = sorted(set(int(v) for v in levels))
    for L in levels:
        _check_level(L, dfield.n_decoders)
    mask = 0
    for L in levels:
        mask |= 1 << (L - 1)
    pts = np.ascontiguousarray(np.atleast_2d(np.asarray(x, dtype=np.float64)))
    n, ncols = len(pts), len(levels)
    out = np.empty((n, ncols), dtype=np.float64)
    if n == 0:
        return out
    if pts.shape[1] != 3:
        raise StructuralError("points must be (n, 3)")
    dev = _lib.device()
    st = _staging(dev, ncols)
    cur = torch.cuda.current_stream(dev)
    cnt = _Counters()
    lo = torch.full((1,), np.inf, dtype=torch.float64, device=dev)
    hi = torch.full((1,), -np.inf, dtype=torch.float64, device=dev)
    args = _lib.NgQueryArgs(mask, -1, 0, 0, 0.0)
    ev_h2d = [torch.cuda.Event(), torch.cuda.Event()]
    ev_k = [torch.cuda.Event(), torch.cuda.Event()]
    ev_d2h = [torch.cuda.Event(), torch.cuda.Event()]
    used = [False, False]
    st.copy.wait_stream(cur)  # the caller's queued work (e.g. a field update) first
    pending = None

    def drain(p):
        s, a, b = p
        ev_d2h[s].synchronize()
        torch.from_numpy(out[a:b]).copy_(st.pin_out[s][:b - a])

    for i, a in enumerate(range(0, n, HOST_CHUNK)):
        b = min(a + HOST_CHUNK, n)
        m, s = b - a, i % 2
        if used[s]:
            ev_h2d[s].synchronize()  # pin_in[s] was read by its last H2D
        st.pin_in[s][:m].copy_(torch.from_numpy(pts[a:b]))
        with torch.cuda.stream(st.copy):
            if used[s]:
                st.copy.wait_event(ev_k[s])  # d_in[s] was read by its last kernel
            st.d_in[s][:m].copy_(st.pin_in[s][:m], non_blocking=True)
            ev_h2d[s].record(st.copy)
        cur.wait_event(ev_h2d[s])
        if used[s]:
            cur.wait_event(ev_d2h[s])  # d_out[s] was read by its last D2H
        d_in, d_out = st.d_in[s][:m], st.d_out[s][:m]
        mn, mx = torch.aminmax(d_in)
        torch.minimum(lo, mn, out=lo)
        torch.maximum(hi, mx, out=hi)
        call("ng_query", svo.device.ref(), dfield.ref(), ctypes.byref(args), ptr(d_in), m, ptr(d_out), cnt.ptr(),
             stream_ptr())
        ev_k[s].record(cur)
        with torch.cuda.stream(st.copy):
            st.copy.wait_event(ev_k[s])
            st.pin_out[s][:m].copy_(d_out, non_blocking=True)
            ev_d2h[s].record(st.copy)
        used[s] = True
        if pending is not None:
            drain(pending)  # the previous chunk, while this one runs
        pending = (s, a, b)
    drain(pending)
    cur.wait_stream(st.copy)
    if float(lo.item()) < DOMAIN_MIN or float(hi.item()) > DOMAIN_MAX:
        raise StructuralError("point outside the domain box")
    c = cnt.host()
    if c[3]:
        raise OctfieldError("non-finite decoder input")
    if counter is not None:
        counter.add(c)
    return out


# host parameter arrays -> the fields holding a device copy of them, so an
# in-place update through the API (trainer.adam_step) drops stale copies
_WATCHED: dict = {}


def _watch(fld) -> None:
    arrays = [fld.Z] + [getattr(d, k) for d in fld.decoders for k in ("W1", "b1", "W2", "b2")]
    for a in arrays:
        _WATCHED.setdefault(id(a), weakref.WeakSet()).add(fld)


def invalidate_arrays(arrays) -> None:
    """Drop the device copies of every field that holds one of `arrays`
    (after they were changed in place)."""
    for a in arrays:
        for fld in list(_WATCHED.get(id(a), ())):
            fld.invalidate()


@dataclass(eq=False)
class NeuralField:
    """Octree plus parameters (field.py:242-269). The device copy of the
    parameters is made on first use; call `invalidate()` after editing Z or
    the decoders in place."""

    svo: SparseVoxelOctree
    Z: np.ndarray
    decoders: list
    _device: DeviceField | None = field(default=None, repr=False, compare=False)

    @property
    def max_level(self) -> int:
        return self.svo.max_level

    @property
    def feature_dim(self) -> int:
        return int(np.shape(self.Z)[1])

    @property
    def hidden_dim(self) -> int:
        return self.decoders[0].W1.shape[0]

    @property
    def device(self) -> DeviceField:
        if self._device is None:
            self._device = DeviceField(self.Z, self.decoders)
            _watch(self)
        return self._device

    def invalidate(self) -> None:
        self._device = None

    def predict(self, x, L: int, counter: EvalCounter | None = None):
        return predict(self.svo, self.Z, self.decoders, x, L, counter, self.device)

    def blend(self, x, L_tilde: float, counter: EvalCounter | None = None):
        return blend(self.svo, self.Z, self.decoders, x, L_tilde, counter, self.device)

    def forward(self, x, L: int):
        return forward(self.svo, self.Z, self.decoders, x, L, self.device)

    def forward_levels(self, x, levels):
        return _host_query(self.svo, self.device, x, levels)


def new_field(svo: SparseVoxelOctree, m: int = FEATURE_DIM, h: int = HIDDEN_DIM, seed: int = 0) -> NeuralField:
    """Freshly initialised field (field.py:272-283)."""
    return NeuralField(svo, init_features(svo, m, seed), init_decoders(svo.max_level, m, h, seed + 1))
