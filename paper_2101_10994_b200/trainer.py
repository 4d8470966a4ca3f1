"""Optimisation of the field against a ground-truth oracle, on the GPU.

Drop-in for octfield.trainer (trainer.py:1-296). Each epoch draws a fresh
2:2:1 surface / near / uniform mixture (sampling.py, host data loader),
shuffles it, uploads it once, and runs every mini-batch's loss, backward
pass and Adam step on the device (csrc/train.cu, ng_train_epoch) with
float64 master weights like the reference. The per-batch step is
deterministic: gradients are reduced in a fixed order without floating-point
atomics, so the trained parameters are bit-identical across runs (the
reference's guarantee across worker counts, trainer.py:8-10).
"""

from __future__ import annotations

import csv
import ctypes
import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream_ptr
from .errors import ConfigError, TrainingDiverged, StructuralError
from .field import (
    Decoder,
    DecoderGrads,
    FieldGradients,
    LevelInterp,
    NeuralField,
    _dev_points,
    invalidate_arrays,
    decoder_stride,
    trilinear,
)
from .sampling import SampleSet, build_epoch_set

SCHEDULES = ("joint", "progressive", "frozen_decoder")

ADAM_BETA1 = 0.9
ADAM_BETA2 = 0.999
ADAM_EPS = 1e-8


@dataclass
class TrainConfig:
    """trainer.py:36-59 (same fields and validation)."""

    epochs: int
    points_per_epoch: int = 500_000
    batch_size: int = 512
    learning_rate: float = 0.001
    schedule: str = "joint"
    progressive_interval: int = 100
    rng_seed: int = 0
    workers: int = 1
    log_path: str | None = None
    checkpoint_every: int = 0
    checkpoint_dir: str | None = None

    def __post_init__(self):
        if self.epochs < 0:
            raise ConfigError("epochs must be >= 0")
        for name in ("points_per_epoch", "batch_size", "progressive_interval", "workers"):
            if getattr(self, name) < 1:
                raise ConfigError(f"{name} must be positive")
        if self.learning_rate <= 0.0:
            raise ConfigError("learning_rate must be positive")
        if self.schedule not in SCHEDULES:
            raise ConfigError(f"schedule must be one of {SCHEDULES}")
        if self.checkpoint_every < 0:
            raise ConfigError("checkpoint_every must be >= 0")
        if self.checkpoint_every and not self.checkpoint_dir:
            raise ConfigError("checkpoint_every needs checkpoint_dir")


# ----------------------------------------------------------------- device state

def _pack64(decoders: list, m: int, h: int) -> np.ndarray:
    stride = decoder_stride(h)
    buf = np.zeros((len(decoders), stride), dtype=np.float64)
    for i, d in enumerate(decoders):
        W1 = np.asarray(d.W1, dtype=np.float64)
        if W1.shape != (h, 3 + m):
            raise StructuralError("decoders must share (h, 3 + m) shapes")
        blk = buf[i, :h * 36].reshape(h, 36)
        blk[:, :3 + m] = W1
        blk[:, 35] = np.asarray(d.b1, dtype=np.float64).ravel()
        buf[i, h * 36:h * 37] = np.asarray(d.W2, dtype=np.float64).ravel()
        buf[i, h * 37] = float(np.asarray(d.b2, dtype=np.float64).ravel()[0])
    return buf


def _unpack64(buf: np.ndarray, m: int, h: int, i: int) -> Decoder:
    blk = buf[i, :h * 36].reshape(h, 36)
    return Decoder(blk[:, :3 + m].copy(), blk[:, 35].copy(), buf[i, h * 36:h * 37].reshape(1, h).copy(),
                   buf[i, h * 37:h * 37 + 1].copy())


class DeviceTrainState:
    """fp64 master parameters and Adam moments in HBM (ng_train_params):
    Z padded to 32 channels, decoders packed as W1b[h][36] | W2 | b2."""

    def __init__(self, svo, Z, decoders: list, moments: bool = True):
        dev = _lib.device()
        Zn = np.asarray(Z, dtype=np.float64)
        if Zn.ndim != 2 or Zn.shape[1] > _lib.FEAT_PAD:
            raise StructuralError(f"feature volume of shape {Zn.shape} not supported")
        if len(decoders) != svo.max_level:
            raise StructuralError("one decoder per level is required")
        self.svo = svo
        self.m = Zn.shape[1]
        self.h = decoders[0].W1.shape[0]
        self.n_dec = len(decoders)
        self.C = Zn.shape[0]
        self.stride = decoder_stride(self.h)
        Zp = np.zeros((self.C, _lib.FEAT_PAD), dtype=np.float64)
        Zp[:, :self.m] = Zn
        self.Z = torch.from_numpy(Zp).to(dev)
        self.dec = torch.from_numpy(_pack64(decoders, self.m, self.h)).to(dev)
        if moments:
            self.Zm, self.Zv = torch.zeros_like(self.Z), torch.zeros_like(self.Z)
            self.decm, self.decv = torch.zeros_like(self.dec), torch.zeros_like(self.dec)
            self.Zlast = torch.zeros(self.C, dtype=torch.int32, device=dev)
        else:
            self.Zm = self.Zv = self.decm = self.decv = self.Zlast = None
        s = _lib.NgTrainParams()
        s.Z, s.Zm, s.Zv, s.Zlast = ptr(self.Z), ptr(self.Zm), ptr(self.Zv), ptr(self.Zlast)
        s.dec, s.decm, s.decv = ptr(self.dec), ptr(self.decm), ptr(self.decv)
        s.m, s.h, s.n_decoders, s.dec_stride = self.m, self.h, self.n_dec, self.stride
        s.corner_count = self.C
        self.struct = s
        self._ws = None
        self._ws_cap = 0

    def workspace(self, batch_capacity: int):
        if batch_capacity > self._ws_cap:
            nb = _lib.lib().ng_train_workspace_bytes(self.svo.device.ref(), batch_capacity, self.h, self.n_dec,
                                                     self.C, self.stride)
            self._ws = torch.zeros(int(nb), dtype=torch.uint8, device=self.Z.device)  # counters start at zero
            self._ws_cap = batch_capacity
        return self._ws

    # -- host views
    def Z_numpy(self) -> np.ndarray:
        return self.Z[:, :self.m].cpu().numpy().copy()

    def decoders_numpy(self) -> list:
        buf = self.dec.cpu().numpy()
        return [_unpack64(buf, self.m, self.h, i) for i in range(self.n_dec)]

    # -- one batch in gradient mode (loss_batch / backward)
    def gradients(self, pts: np.ndarray, dist, active_mask: int, denom: float, grads: FieldGradients,
                  upstream=None) -> np.ndarray:
        n = len(pts)
        sums = torch.zeros(self.n_dec, dtype=torch.float64, device=self.Z.device)
        if n == 0:
            return sums.cpu().numpy()
        dev = self.Z.device
        dp = _dev_points(pts)
        dd = torch.from_numpy(np.ascontiguousarray(dist, dtype=np.float64)).to(dev) if dist is not None else None
        du = torch.from_numpy(np.ascontiguousarray(upstream, dtype=np.float64)).to(dev) if upstream is not None else None
        gZ = torch.zeros((self.C, _lib.FEAT_PAD), dtype=torch.float64, device=dev)
        gZ[:, :self.m] = torch.from_numpy(np.asarray(grads.dZ, dtype=np.float64)).to(dev)
        held = [g if g is not None else DecoderGrads(np.zeros((self.h, 3 + self.m)), np.zeros(self.h),
                                                     np.zeros((1, self.h)), np.zeros(1)) for g in grads.decoders]
        gD = torch.from_numpy(_pack64(held, self.m, self.h)).to(dev)
        touched = torch.tensor([int(g is not None) for g in grads.decoders], dtype=torch.int32, device=dev)
        status = torch.zeros(1, dtype=torch.int64, device=dev)
        ws = self.workspace(n)
        st = _lib.NgTrainStep(active_mask, 0, 1, 0, float(denom), 0.0, 0, None, 0)
        call("ng_train_batch", self.svo.device.ref(), ctypes.byref(self.struct), ctypes.byref(st), ptr(dp), ptr(dd),
             ptr(du), n, self._ws_cap, ptr(ws), ws.numel(), ptr(sums), ptr(gZ), ptr(gD), ptr(touched), None,
             ptr(status), stream_ptr())
        grads.dZ[...] = gZ[:, :self.m].cpu().numpy()
        buf = gD.cpu().numpy()
        for i, t in enumerate(touched.cpu().numpy()):
            if t:
                d = _unpack64(buf, self.m, self.h, i)
                grads.decoders[i] = DecoderGrads(d.W1, d.b1, d.W2, d.b2)
        return sums.cpu().numpy()

    # -- ForwardCache contents of forward(x, L) (field.py:321-357)
    def export(self, pts: np.ndarray, L: int) -> dict:
        n = len(pts)
        dev = self.Z.device
        ids = torch.full((n, L, 8), -1, dtype=torch.int32, device=dev)
        w = torch.zeros((n, L, 8), dtype=torch.float64, device=dev)
        psi = torch.zeros((n, L, _lib.FEAT_PAD), dtype=torch.float64, device=dev)
        pre = torch.zeros((n, self.h), dtype=torch.float64, device=dev)
        inp = torch.zeros((n, 36), dtype=torch.float64, device=dev)
        if n:
            dp = _dev_points(pts)
            # ng_train_export lays its workspace out for a capacity of exactly n
            nb = _lib.lib().ng_train_workspace_bytes(self.svo.device.ref(), n, self.h, self.n_dec, self.C,
                                                     self.stride)
            ws = torch.zeros(int(nb), dtype=torch.uint8, device=dev)
            call("ng_train_export", self.svo.device.ref(), ctypes.byref(self.struct), L, ptr(dp), n, ptr(ws),
                 ws.numel(), ptr(ids), ptr(w), ptr(psi), ptr(pre), ptr(inp), stream_ptr())
        ids_h, w_h, psi_h = ids.cpu().numpy(), w.cpu().numpy(), psi.cpu().numpy()
        recs = []
        anyl = np.zeros(n, dtype=bool)
        for lv in range(1, L + 1):
            mask = ids_h[:, lv - 1, 0] >= 0
            anyl |= mask
            recs.append(LevelInterp(lv, mask, ids_h[mask, lv - 1], w_h[mask, lv - 1], psi_h[:, lv - 1, :self.m]))
        rows = np.flatnonzero(anyl)
        return {"recs": recs, "rows": rows, "inp": inp.cpu().numpy()[rows, :3 + self.m],
                "pre": pre.cpu().numpy()[rows]}


# ----------------------------------------------------------------- loss / Adam

def _active(active_levels, max_level: int) -> list:
    active = sorted(set(int(L) for L in active_levels))
    if not active:
        raise ConfigError("active level set is empty")
    if active[0] < 1 or active[-1] > max_level:
        raise ConfigError(f"active levels {active} outside 1..{max_level}")
    return active


def loss_batch(fld: NeuralField, samples: SampleSet, active_levels, grads: FieldGradients | None = None,
               denom: int | None = None, predict_fn=None):
    """Squared-error loss summed across active levels (trainer.py:106-144).

    Returns (loss, grads, level_sums). A point skips a level's term when no
    voxel at that level contains it. predict_fn(points, L) substitutes the
    predictor for loss-only checks (gradients are then skipped)."""
    active = _active(active_levels, fld.max_level)
    pts = np.asarray(samples.points, dtype=np.float64)
    d = np.asarray(samples.distances, dtype=np.float64)
    n = len(samples) if denom is None else denom
    level_sums = np.zeros(fld.max_level)
    if predict_fn is not None:
        for L in active:
            out = np.asarray(predict_fn(pts, L), dtype=np.float64)
            _, mask = trilinear(fld.svo, fld.Z, pts, L)
            resid = np.where(mask, out - d, 0.0)
            level_sums[L - 1] = float(resid @ resid)
        return float(level_sums[np.array(active) - 1].sum() / n), None, level_sums
    if grads is None:
        grads = FieldGradients.zeros(fld.Z, fld.max_level)
    mask = 0
    for L in active:
        mask |= 1 << (L - 1)
    st = DeviceTrainState(fld.svo, fld.Z, fld.decoders, moments=False)
    level_sums = st.gradients(pts, d, mask, n, grads)
    loss = float(level_sums[np.array(active) - 1].sum() / n)
    return loss, grads, level_sums


@dataclass
class AdamState:
    """First/second moments mirroring the parameter dict (trainer.py:62-84)."""

    m: dict
    v: dict
    step: int = 0
    beta1: float = ADAM_BETA1
    beta2: float = ADAM_BETA2
    eps: float = ADAM_EPS

    @classmethod
    def for_params(cls, params: dict) -> "AdamState":
        return cls(m={k: np.zeros(p.shape) for k, p in params.items()},
                   v={k: np.zeros(p.shape) for k, p in params.items()})


def adam_step(params: dict, grads: dict, state: AdamState, lr: float):
    """One bias-corrected Adam update in place (trainer.py:87-103); each
    array is updated by the device kernel (ng_adam_step). Parameters without
    a gradient entry are untouched."""
    state.step += 1
    c1 = 1.0 - state.beta1 ** state.step
    c2 = 1.0 - state.beta2 ** state.step
    dev = _lib.device()
    for name, g in grads.items():
        p = torch.from_numpy(np.ascontiguousarray(params[name], dtype=np.float64)).to(dev)
        m = torch.from_numpy(np.ascontiguousarray(state.m[name], dtype=np.float64)).to(dev)
        v = torch.from_numpy(np.ascontiguousarray(state.v[name], dtype=np.float64)).to(dev)
        gd = torch.from_numpy(np.ascontiguousarray(g, dtype=np.float64)).to(dev)
        bad = torch.zeros(1, dtype=torch.int64, device=dev)
        call("ng_adam_step", ptr(p), ptr(m), ptr(v), ptr(gd), p.numel(), float(lr), c1, c2, ptr(bad), stream_ptr())
        if int(bad.item()):
            raise TrainingDiverged(f"non-finite gradient for {name}")
        params[name][...] = p.cpu().numpy().reshape(np.shape(params[name]))
        state.m[name][...] = m.cpu().numpy().reshape(np.shape(g))
        state.v[name][...] = v.cpu().numpy().reshape(np.shape(g))
        # fields holding a device copy of this array re-upload on next use
        invalidate_arrays([params[name]])
    return params, state


@dataclass
class EpochStats:
    epoch: int
    level_losses: np.ndarray  # (max_level,); nan where the level was inactive
    seconds: float


def active_levels_for(schedule: str, epoch: int, interval: int, max_level: int) -> list:
    """Level set of one epoch (trainer.py:154-162)."""
    if schedule == "progressive":
        n = min(1 + epoch // interval, max_level)
        return list(range(max_level - n + 1, max_level + 1))
    return list(range(1, max_level + 1))


# ----------------------------------------------------------------- training

class DeviceTrainer:
    """The epoch loop's device half: parameters, moments, workspace and the
    Adam step counter persist across epochs in HBM."""

    def __init__(self, fld: NeuralField, batch_size: int, flush_every: int = 32):
        self.state = DeviceTrainState(fld.svo, fld.Z, fld.decoders, moments=True)
        self.batch_size = batch_size
        self.flush_every = flush_every
        self.step = 0
        dev = self.state.Z.device
        self.level_sums = torch.zeros(self.state.n_dec, dtype=torch.float64, device=dev)
        self.status = torch.zeros(1, dtype=torch.int64, device=dev)
        self.adam_c = torch.zeros(0, dtype=torch.float64, device=dev)

    def _bias_table(self, upto: int) -> None:
        """(1 - beta1^t, 1 - beta2^t) for steps 1..upto, computed like
        adam_step (trainer.py:92-93) and kept on the device."""
        have = self.adam_c.numel() // 2
        if upto <= have:
            return
        upto = max(upto, 2 * have)
        c = np.empty((upto, 2), dtype=np.float64)
        for t in range(1, upto + 1):
            c[t - 1, 0] = 1.0 - ADAM_BETA1 ** t
            c[t - 1, 1] = 1.0 - ADAM_BETA2 ** t
        self.adam_c = torch.from_numpy(c.ravel()).to(self.state.Z.device)

    def run_epoch(self, pts_dev: torch.Tensor, dist_dev: torch.Tensor, active: list, update_decoders: bool,
                  lr: float) -> None:
        """Enqueue every mini-batch of one epoch (asynchronous)."""
        st = self.state
        n = pts_dev.shape[0]
        mask = 0
        for L in active:
            mask |= 1 << (L - 1)
        self.level_sums.zero_()
        ws = st.workspace(self.batch_size)
        n_batches = (n + self.batch_size - 1) // self.batch_size
        self._bias_table(self.step + n_batches)
        call("ng_train_epoch", st.svo.device.ref(), ctypes.byref(st.struct), ptr(pts_dev), ptr(dist_dev), n,
             self.batch_size, mask, int(update_decoders), float(lr), self.step, ptr(self.adam_c),
             int(self.flush_every), ptr(ws), ws.numel(), ptr(self.level_sums), ptr(self.status), stream_ptr())
        self.step += n_batches

    def diverged_at(self) -> int:
        """-1, or the start row of the first batch that diverged."""
        return int(self.status.item()) - 1

    def field(self, svo) -> NeuralField:
        return NeuralField(svo, self.state.Z_numpy(), self.state.decoders_numpy())


def train(oracle, fld: NeuralField, config: TrainConfig):
    """Optimise a copy of the field; returns (trained field, epoch stats)
    (trainer.py:165-251). The returned field holds float64 master weights."""
    work_Z = np.asarray(fld.Z, dtype=np.float64).copy()
    work_decs = [d.astype(np.float64) for d in fld.decoders]
    history: list = []
    if config.epochs == 0:
        return NeuralField(fld.svo, work_Z, work_decs), history
    trainer = DeviceTrainer(NeuralField(fld.svo, work_Z, work_decs), config.batch_size)
    update_decoders = config.schedule != "frozen_decoder"
    dev = trainer.state.Z.device
    log_fh = open(config.log_path, "w", newline="") if config.log_path else None
    try:
        writer = None
        if log_fh is not None:
            writer = csv.writer(log_fh)
            writer.writerow(["epoch"] + [f"loss_l{L}" for L in range(1, fld.max_level + 1)] + ["seconds"])
        for epoch in range(config.epochs):
            t0 = time.perf_counter()
            seeds = np.random.SeedSequence([config.rng_seed, epoch]).generate_state(2)
            samples = build_epoch_set(oracle, config.points_per_epoch, int(seeds[0]))
            perm = np.random.default_rng(int(seeds[1])).permutation(len(samples))
            pts = torch.from_numpy(np.ascontiguousarray(samples.points[perm])).to(dev)
            dist = torch.from_numpy(np.ascontiguousarray(samples.distances[perm])).to(dev)
            active = active_levels_for(config.schedule, epoch, config.progressive_interval, fld.max_level)
            trainer.run_epoch(pts, dist, active, update_decoders, config.learning_rate)
            bad = trainer.diverged_at()
            if bad >= 0:
                raise TrainingDiverged(f"epoch {epoch}, batch at {bad}: non-finite loss or gradient")
            sums = trainer.level_sums.cpu().numpy()
            losses = np.full(fld.max_level, np.nan)
            idx = np.array(active) - 1
            losses[idx] = sums[idx] / len(samples)
            stats = EpochStats(epoch, losses, time.perf_counter() - t0)
            history.append(stats)
            if writer is not None:
                writer.writerow([epoch] + [f"{x:.8g}" for x in losses] + [f"{stats.seconds:.3f}"])
                log_fh.flush()
            if config.checkpoint_every and (epoch + 1) % config.checkpoint_every == 0:
                from . import modelio
                path = os.path.join(config.checkpoint_dir, f"checkpoint_epoch{epoch + 1}.nsdf")
                modelio.save_model(path, trainer.field(fld.svo))
    finally:
        if log_fh is not None:
            log_fh.close()
    return trainer.field(fld.svo), history
