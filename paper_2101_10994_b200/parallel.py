"""Multi-GPU frames: image bands sharded across ranks, framebuffer gathered
over NCCL (BASELINE.json configs[3] / [4]).

One process per GPU. Rays are independent (render.py:389-394 already
shards them), so each rank renders the bands b with b % world == rank
(interleaved 8-row bands balance the costlier silhouette rows) with its own
replica of the octree and field, then the colour (and on request depth,
hit and the other per-pixel outputs) tiles are gathered with one NCCL
collective per output -- to one rank (`dst`) or to all -- and assembled.
A frame's ranks also agree on reruns after a capacity overflow (a one-int
all-reduce). There is no other data-path exchange.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._lib import call, ptr, stream_ptr
from .errors import ConfigError, OctfieldError
from .render import (prepare_presum, Camera, RenderConfig, RenderSession, _batch_cfg, band_rows_of, camera_structs,
                     resolve_config, resolve_lod)

DEFAULT_BAND_ROWS = 8


def band_layout(height: int, world: int, band_rows: int = DEFAULT_BAND_ROWS) -> list:
    """Global rows owned by each rank, in local order."""
    return [band_rows_of(height, band_rows, world, r) for r in range(world)]


def assemble(gathered: torch.Tensor, layout: list, height: int) -> torch.Tensor:
    """Scatter per-rank band tiles back into image order.

    gathered: (world, max_rows, ...) as produced by all_gather_into_tensor of
    row-padded local tiles; returns (height, ...)."""
    world = gathered.shape[0]
    out = gathered.new_empty((height,) + tuple(gathered.shape[2:]))
    for r in range(world):
        rows = layout[r]
        if len(rows):
            idx = torch.as_tensor(rows, dtype=torch.long, device=gathered.device)
            out.index_copy_(0, idx, gathered[r, :len(rows)])
    return out


def _staged(t: torch.Tensor, group) -> bool:
    """gloo moves CPU tensors only: CUDA tiles are staged through the host."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def gather_tiles(local: torch.Tensor, layout: list, height: int, group=None, dst: int | None = None):
    """Gather row-padded local tiles (rows, ...) and assemble the image.

    dst=None all-gathers (every rank gets the image); dst=r gathers to rank
    r only (the other ranks return None). One collective either way."""
    world = dist.get_world_size(group)
    max_rows = max(len(rows) for rows in layout)
    padded = local.new_zeros((max_rows,) + tuple(local.shape[1:]))
    padded[:local.shape[0]] = local
    dev = local.device
    if _staged(local, group):
        padded = padded.cpu()
    tail = tuple(local.shape[1:])
    if dst is None:
        flat = padded.new_empty((world * max_rows,) + tail)
        dist.all_gather_into_tensor(flat, padded, group=group)
        return assemble(flat.view((world, max_rows) + tail), layout, height).to(dev)
    rank = dist.get_rank(group)
    parts = [padded.new_empty(padded.shape) for _ in range(world)] if rank == dst else None
    dist.gather(padded, parts, dst=dst, group=group)
    if rank != dst:
        return None
    return assemble(torch.stack(parts), layout, height).to(dev)


def gather_frames(local: torch.Tensor, layout: list, height: int, group=None, dst: int | None = None):
    """K frames' local band rows (K, rows, ...) -> (K, height, ...) images in
    one collective: the frames ride along as a trailing dimension of each
    row, so the rank layout and the assembly are `gather_tiles`'s."""
    img = gather_tiles(local.transpose(0, 1).contiguous(), layout, height, group, dst)
    return None if img is None else img.transpose(0, 1)


class TiledRenderer:
    """Renders frames of one camera size cooperatively across the ranks of
    the default process group (NCCL). With `batch` > 1, `enqueue` /
    `render_batch` take up to that many cameras per launch sequence (each
    rank renders its bands of every frame in one traversal and one march,
    ng_render_batch), and the frames' tiles are gathered in one collective."""

    def __init__(self, fld, width: int, height: int, band_rows: int = DEFAULT_BAND_ROWS, group=None,
                 batch: int = 1):
        self.fld = fld
        self.width, self.height = width, height
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.band_rows = band_rows
        self.layout = band_layout(height, self.world, band_rows)
        self.local_rows = len(self.layout[self.rank])
        if not 1 <= batch <= _lib.MAX_BATCH:
            raise ConfigError(f"batch must be 1..{_lib.MAX_BATCH}, got {batch}")
        self.batch = batch
        self.frames = 1  # frames in the last launch
        self.sess = RenderSession(fld, width, max(self.local_rows, 1),
                                  n_rays=max(self.local_rows * width, 1) * batch)
        self.frame = self.sess.new_frame()

    def enqueue(self, camera, cfg) -> None:
        """Launch this rank's bands of one camera or of a list of up to
        `batch` cameras (no host sync)."""
        cams = [camera] if isinstance(camera, Camera) else list(camera)
        if not 1 <= len(cams) <= self.batch:
            raise ConfigError(f"this renderer takes 1..{self.batch} cameras per launch, got {len(cams)}")
        cs = camera_structs([c.band_struct(self.band_rows, self.world, self.rank) for c in cams])
        self.frames = len(cams)
        fs = self.sess.frame_struct(self.frame)
        fstruct = prepare_presum(self.fld, cfg)
        if self.local_rows:
            call("ng_render_batch", self.fld.svo.device.ref(), ctypes.byref(fstruct), ctypes.byref(cfg),
                 cs, len(cs), ctypes.byref(fs), ctypes.byref(self.sess.ws), ptr(self.sess.stats),
                 stream_ptr())

    # per-pixel outputs a frame can gather: name -> trailing shape
    _FIELDS = {"color": (3,), "t": (), "hit": (), "normal": (3,), "normal_ok": (), "iterations": (), "evals": ()}

    def _local(self, name: str, frames: int = 1) -> torch.Tensor:
        """(local_rows, width, ...) of frame 0, or with frames > 1 the
        first `frames` frames' rows as (frames, local_rows, width, ...)."""
        tail = self._FIELDS[name]
        n = self.local_rows * self.width
        v = self.frame[name][:n * frames].reshape((frames, self.local_rows, self.width) + tail)
        return v[0] if frames == 1 else v

    def gather(self, fields=("color",), dst: int | None = None, frames: int | None = None) -> dict:
        """The frame's per-pixel outputs assembled to (height, width, ...)
        device tensors: on every rank (dst=None, all-gather) or on rank dst
        only (gather; the other ranks get an empty dict). One collective per
        field (colour, plus depth / hit on request). With
        `frames` (default: 1 after a single camera, else the last launch's
        frames) > 1, each field is (frames, height, width, ...), every
        frame's tiles moving in the same collective."""
        k = frames if frames is not None else self.frames
        out = {}
        for name in fields:
            local = self._local(name, k)
            if self.world == 1:
                out[name] = local
                continue
            if k == 1:
                img = gather_tiles(local, self.layout, self.height, self.group, dst)
            else:
                img = gather_frames(local, self.layout, self.height, self.group, dst)
            if img is not None:
                out[name] = img
        return out

    def gather_color(self, dst: int | None = None):
        """(height, width, 3) uint8 image (None on ranks other than dst)."""
        return self.gather(("color",), dst).get("color")

    def render(self, camera: Camera, config: RenderConfig, fields=None, dst: int | None = None):
        """One frame across the ranks. Returns (image (H, W, 3) uint8 device
        tensor, visible, evals), or with `fields` (names of per-pixel
        outputs: color, t, hit, normal, ...) a dict of them in place of the
        image; with dst, only rank dst receives the images."""
        lod = resolve_lod(camera, self.fld, config)
        cfg = resolve_config(self.fld, config, lod)
        return self._render(camera, cfg, fields, dst)

    def render_batch(self, cameras, config: RenderConfig, fields=None, dst: int | None = None):
        """Up to `batch` frames across the ranks in one launch sequence per
        rank. Returns (images (K, H, W, 3) uint8, visible, evals) with the
        batch's totals, or with `fields` a dict of (K, H, W, ...) outputs;
        each frame equals `render`'s for its camera."""
        cams = list(cameras)
        _, cfg = _batch_cfg(cams, self.fld, config)
        return self._render(cams, cfg, fields, dst)

    def _render(self, camera, cfg, fields, dst):
        n_levels = cfg.trace_level + self.fld.svo.device.n_virtual
        self.reruns = 0
        while True:
            self.enqueue(camera, cfg)
            st = self.sess.read_stats()
            # every rank reruns when any rank overflowed (the frame's ranks
            # must agree on the number of collectives)
            again = torch.tensor([1 if st.overflow else 0], device=_lib.device())
            if self.world > 1:
                if _staged(again, self.group):
                    a = again.cpu()
                    dist.all_reduce(a, group=self.group)
                    again = a
                else:
                    dist.all_reduce(again, group=self.group)
            if st.overflow:
                self.sess.grow(st, n_levels)
            if int(again.item()) == 0:
                break
            self.reruns += 1
        if st.counters.evals_missing_level or st.counters.nonfinite_inputs:
            raise OctfieldError("decoder ran outside the queried level's voxels or on non-finite input")
        imgs = self.gather(fields or ("color",), dst)
        counts = torch.tensor([st.visible, st.counters.decoder_evals], dtype=torch.int64, device=_lib.device())
        if self.world > 1:
            if _staged(counts, self.group):
                c = counts.cpu()
                dist.all_reduce(c, group=self.group)
                counts = c
            else:
                dist.all_reduce(counts, group=self.group)
        if fields is None:
            imgs = imgs.get("color")
        return imgs, int(counts[0].item()), int(counts[1].item())
