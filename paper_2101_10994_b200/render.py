"""Sphere tracing of the octree field on the GPU, and image output.

Drop-in for octfield.render (render.py:1-448). A frame is one C-ABI call
(`ng_render_frame`): device ray generation (bit-exact with Camera.rays),
the breadth-first traversal, the persistent-lane sphere-trace march, the
central-difference normals with Lambert shading fused in, and frame
statistics -- no host synchronisation until the caller reads a result.
`FrameBuffer` fields are device tensors materialised as numpy on access.
"""

from __future__ import annotations

import os
import threading

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream_ptr
from .errors import ConfigError, OctfieldError, StructuralError
from .field import EvalCounter, NeuralField, _Counters, _dev_points, _run_exact
from .octree import DOMAIN_MAX, DOMAIN_MIN
from .traversal import RayBundle, RayVoxelPairList, device_rays, ray_segments

_RAY_SHARD = 8192  # kept for API parity; the device path has no shards


@dataclass
class Camera:
    """Pinhole camera (render.py:43-88)."""

    position: np.ndarray
    look_at: np.ndarray
    up: np.ndarray
    fov_y_deg: float
    width: int
    height: int

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64)
        self.look_at = np.asarray(self.look_at, dtype=np.float64)
        self.up = np.asarray(self.up, dtype=np.float64)
        if not 0.0 < self.fov_y_deg < 180.0:
            raise ConfigError("vertical FOV must be in (0, 180) degrees")
        if self.width < 1 or self.height < 1:
            raise ConfigError("image dimensions must be positive")
        fwd = self.look_at - self.position
        if np.linalg.norm(fwd) < 1e-12:
            raise ConfigError("camera position and look_at coincide")
        if np.linalg.norm(np.cross(fwd, self.up)) < 1e-12:
            raise ConfigError("up vector is parallel to the view direction")

    def basis(self):
        fwd = self.look_at - self.position
        fwd = fwd / np.linalg.norm(fwd)
        right = np.cross(fwd, self.up)
        right = right / np.linalg.norm(right)
        true_up = np.cross(right, fwd)
        return fwd, right, true_up

    def _key(self):
        return (self.position.tobytes(), self.look_at.tobytes(), self.up.tobytes(), float(self.fov_y_deg),
                int(self.width), int(self.height))

    def struct(self) -> _lib.NgCamera:
        """The C camera (basis in fp64), cached on the camera for its current
        parameters; callers get their own copy."""
        key = self._key()
        cached = self.__dict__.get("_struct_cache")
        if cached is None or cached[0] != key:
            cached = (key, self._make_struct())
            self.__dict__["_struct_cache"] = cached
        return _lib.NgCamera.from_buffer_copy(cached[1])

    def _make_struct(self) -> _lib.NgCamera:
        fwd, right, up = self.basis()
        c = _lib.NgCamera()
        for a in range(3):
            c.position[a] = float(self.position[a])
            c.fwd[a] = float(fwd[a])
            c.right[a] = float(right[a])
            c.up[a] = float(up[a])
        c.tan_half = math.tan(math.radians(self.fov_y_deg) / 2.0)
        c.aspect = self.width / self.height
        c.width = int(self.width)
        c.height = int(self.height)
        c.band_rows, c.band_stride, c.band_offset, c.local_rows = int(self.height), 1, 0, int(self.height)
        return c

    def band_struct(self, band_rows: int, stride: int, offset: int) -> _lib.NgCamera:
        """Camera restricted to the image bands owned by one of `stride`
        ranks (bands of `band_rows` rows, band b to rank b % stride)."""
        c = self.struct()
        c.band_rows, c.band_stride, c.band_offset = int(band_rows), int(stride), int(offset)
        c.local_rows = len(band_rows_of(self.height, band_rows, stride, offset))
        return c

    def device_rays(self) -> torch.Tensor:
        n = self.width * self.height
        buf = torch.empty(n * _lib.RAY_BYTES, dtype=torch.uint8, device=_lib.device())
        call("ng_camera_rays", ctypes.byref(self.struct()), ptr(buf), stream_ptr())
        return buf

    def rays(self) -> RayBundle:
        """Primary rays through pixel centres, row-major, row 0 at the top
        (render.py:74-88); generated on the device."""
        raw = self.device_rays().cpu().numpy()
        rec = raw.view(np.float64).reshape(-1, 10)
        return RayBundle(rec[:, 0:3].copy(), rec[:, 3:6].copy())


def band_rows_of(height: int, band_rows: int, stride: int, offset: int) -> np.ndarray:
    """Global image rows of the bands b = offset, offset + stride, ... in order."""
    rows = np.arange(height)
    return rows[(rows // band_rows) % stride == offset]


@dataclass
class RenderConfig:
    """render.py:91-114."""

    delta: float = 0.0003
    max_iters: int = 200
    far_plane: float = 5.0
    lod: float | None = None
    lod_thresholds: list | None = None
    normal_eps: float | None = None
    skip_eps: float = 1e-5
    osc_factor: float = 6.0
    workers: int = 1
    light_dir: tuple = (-0.45, 0.8, -0.55)
    albedo: tuple = (0.82, 0.84, 0.88)
    ambient: float = 0.12
    background: tuple = (0.09, 0.10, 0.13)
    # extension (BASELINE.json configs[4]; not in the reference): secondary
    # shadow rays from p + shadow_offset * n toward the light (default offset
    # 2 * normal_eps, one finest voxel edge); shadowed pixels get the ambient term
    shadows: bool = False
    shadow_offset: float | None = None

    def __post_init__(self):
        if self.shadow_offset is not None and self.shadow_offset <= 0.0:
            raise ConfigError("shadow_offset must be positive")
        for name in ("delta", "far_plane", "skip_eps", "osc_factor"):
            if getattr(self, name) <= 0.0:
                raise ConfigError(f"{name} must be positive")
        if self.max_iters < 1 or self.workers < 1:
            raise ConfigError("max_iters and workers must be positive")
        if self.normal_eps is not None and self.normal_eps <= 0.0:
            raise ConfigError("normal_eps must be positive")


class FrameBuffer:
    """Per-pixel outputs (render.py:117-128). Backed by device tensors; each
    field is copied to the host on first access."""

    _FIELDS = ("hit", "t", "points", "normal", "normal_ok", "iterations", "evals", "color")

    def __init__(self, width, height, dev: dict, camera: Camera | None = None, rays: torch.Tensor | None = None,
                 prefetched: dict | None = None):
        self.width = width
        self.height = height
        self.device = dev
        self._camera = camera
        self._rays = rays
        self._host = {}
        self._pinned = prefetched or {}  # host copies already issued on the stream (pinned)

    def _shape(self, *tail):
        return (self.height, self.width) + tail

    def _get(self, name):
        if name in self._host:
            return self._host[name]
        d = self.device
        if name == "hit":
            v = d["hit"].cpu().numpy().astype(bool).reshape(self._shape())
        elif name == "t":
            v = d["t"].cpu().numpy().reshape(self._shape())
        elif name == "normal":
            v = d["normal"].cpu().numpy().reshape(self._shape(3))
        elif name == "normal_ok":
            v = d["normal_ok"].cpu().numpy().astype(bool).reshape(self._shape())
        elif name == "iterations":
            v = d["iterations"].cpu().numpy().reshape(self._shape())
        elif name == "evals":
            v = d["evals"].cpu().numpy().astype(np.int64).reshape(self._shape())
        elif name == "color":
            src = self._pinned["color"] if "color" in self._pinned else d["color"].cpu()
            v = src.numpy().reshape(self._shape(3))
        elif name == "points":
            n = self.width * self.height
            rays = self._rays if self._rays is not None else self._camera.device_rays()
            out = torch.empty((n, 3), dtype=torch.float64, device=d["t"].device)
            call("ng_hit_points", ptr(rays), ptr(d["hit"]), ptr(d["t"]), n, ptr(out), stream_ptr())
            v = out.cpu().numpy().reshape(self._shape(3))
        else:
            raise AttributeError(name)
        self._host[name] = v
        return v

    def __getattr__(self, name):
        if name in FrameBuffer._FIELDS:
            return self._get(name)
        raise AttributeError(name)

    def __setattr__(self, name, value):
        if name in FrameBuffer._FIELDS:
            self._host[name] = value
        else:
            object.__setattr__(self, name, value)


@dataclass
class FrameReport:
    """render.py:131-137; times are CUDA-event device times."""

    ms_trace: float
    ms_normals: float
    evals: int
    visible: int
    lod: float
    shadowed: int = 0


def select_lod(camera: Camera, svo, thresholds) -> float:
    """Piecewise-linear detail level from the eye-to-region distance (render.py:140-152)."""
    th = np.asarray(thresholds, dtype=np.float64)
    if th.ndim != 1 or len(th) != svo.max_level:
        raise ConfigError(f"need {svo.max_level} distance thresholds")
    if np.any(np.diff(th) <= 0.0):
        raise ConfigError("thresholds must be strictly increasing")
    center = 0.5 * (svo.region.lo + svo.region.hi)
    dist = float(np.linalg.norm(np.asarray(camera.position) - center))
    levels = np.arange(svo.max_level, 0, -1, dtype=np.float64)
    return float(np.interp(dist, th, levels))


def _trace_level(fld: NeuralField, lod: float) -> int:
    return min(int(math.ceil(max(lod, 1.0))), fld.max_level)


def resolve_config(fld: NeuralField, config: RenderConfig, lod: float, eps: float | None = None) -> _lib.NgRenderCfg:
    c = _lib.NgRenderCfg()
    c.delta = float(config.delta)
    c.far_plane = float(config.far_plane)
    c.skip_eps = float(config.skip_eps)
    c.osc_tol = float(config.osc_factor * config.delta)
    c.lod = float(lod)
    if eps is None:
        eps = config.normal_eps if config.normal_eps is not None else 0.5 * fld.svo.voxel_edge(fld.max_level)
    c.normal_eps = float(eps)
    light = np.asarray(config.light_dir, dtype=np.float64)
    light = light / np.linalg.norm(light)
    for a in range(3):
        c.light[a] = float(light[a])
        c.albedo[a] = float(config.albedo[a])
        c.background[a] = float(config.background[a])
    c.ambient = float(config.ambient)
    c.max_iters = int(config.max_iters)
    c.trace_level = _trace_level(fld, lod)
    c.shadows = 1 if getattr(config, "shadows", False) else 0
    off = getattr(config, "shadow_offset", None)
    c.shadow_offset = float(off) if off is not None else 2.0 * c.normal_eps
    return c


_PRESUM = os.environ.get("NG_PRESUM", "1") != "0"


def prepare_presum(fld: NeuralField, cfg: _lib.NgRenderCfg) -> _lib.NgField:
    """The field struct a frame launches with: carrying the presummed
    feature tables of this frame's gather level and output levels (the
    LodPlan of render.cu: blend levels for a fractional lod) when they
    apply; NG_PRESUM=0 keeps the level-by-level gather."""
    if _PRESUM:
        lod = max(float(cfg.lod), 1.0)
        base = int(np.floor(lod))
        if lod - base == 0.0:
            mask, G = 1 << (base - 1), max(base, cfg.trace_level)
        else:
            mask, G = (1 << (base - 1)) | (1 << base), max(base + 1, cfg.trace_level)
        if G == cfg.trace_level:
            return fld.device.presum_struct(fld.svo, G, mask)
    return fld.device.struct


def _lod_split(lod: float):
    L = max(float(lod), 1.0)
    base = int(np.floor(L))
    return base, L - base


def query_field(fld: NeuralField, pts: np.ndarray, lod: float, counter: EvalCounter | None = None) -> np.ndarray:
    """Decode only inside trace-level voxels; elsewhere the empty-space
    value (render.py:155-171)."""
    p = np.atleast_2d(np.asarray(pts, dtype=np.float64))
    lvl = _trace_level(fld, lod)
    if lod > len(fld.decoders):
        raise StructuralError(f"blend level {lod} above max {len(fld.decoders)}")
    base, alpha = _lod_split(lod)
    if alpha == 0.0:
        out = _run_exact(fld.svo, fld.device, _dev_points(p), out_levels=1 << (base - 1), inside_level=lvl,
                         counter=counter)
    else:
        out = _run_exact(fld.svo, fld.device, _dev_points(p), inside_level=lvl, blend_base=base, blend_alpha=alpha,
                         counter=counter)
    return out[:, 0].cpu().numpy()


def _hit_records(final: RayVoxelPairList) -> torch.Tensor:
    n = len(final)
    rec = np.zeros(max(n, 1), dtype=np.dtype([("ray", "<i4"), ("voxel", "<i4"), ("t_enter", "<f8"),
                                              ("t_exit", "<f8")]))
    if n:
        rec["ray"][:n] = final.rays
        rec["voxel"][:n] = final.voxels
        rec["t_enter"][:n] = final.t_enter
        rec["t_exit"][:n] = final.t_exit
    return torch.from_numpy(np.frombuffer(rec.tobytes(), dtype=np.uint8).copy()).to(_lib.device())


def sphere_trace(fld: NeuralField, rays: RayBundle, final: RayVoxelPairList, lod: float, config: RenderConfig,
                 counter: EvalCounter | None = None):
    """March every ray through its voxel list (render.py:174-274).
    Returns (hit, t_hit, iterations, evals)."""
    n = rays.count
    hit = np.zeros(n, dtype=bool)
    t_hit = np.full(n, np.nan)
    iters = np.zeros(n, dtype=np.int32)
    evals = np.zeros(n, dtype=np.int64)
    if len(final) == 0 or n == 0:
        return hit, t_hit, iters, evals
    dev = _lib.device()
    d_rays = device_rays(rays)
    d_hits = _hit_records(final)
    cnt = torch.tensor([len(final)], dtype=torch.int64, device=dev)
    s, e = ray_segments(final, n)
    d_s = torch.from_numpy(s).to(dev)
    d_e = torch.from_numpy(e).to(dev)
    o_hit = torch.empty(n, dtype=torch.uint8, device=dev)
    o_t = torch.empty(n, dtype=torch.float64, device=dev)
    o_it = torch.empty(n, dtype=torch.int32, device=dev)
    o_ev = torch.empty(n, dtype=torch.int32, device=dev)
    cfg = resolve_config(fld, config, max(float(lod), 1.0))
    cfg.trace_level = final.level
    c = _Counters()
    call("ng_sphere_trace", fld.svo.device.ref(), fld.device.ref(), ctypes.byref(cfg), ptr(d_rays), n, ptr(d_hits),
         ptr(cnt), ptr(d_s), ptr(d_e), ptr(o_hit), ptr(o_t), ptr(o_it), ptr(o_ev), c.ptr(), stream_ptr())
    ch = c.host()
    if ch[3]:
        raise OctfieldError("non-finite decoder input")
    if counter is not None:
        counter.add(ch)
    return (o_hit.cpu().numpy().astype(bool), o_t.cpu().numpy(), o_it.cpu().numpy(),
            o_ev.cpu().numpy().astype(np.int64))


def normals(fld: NeuralField, points: np.ndarray, eps: float, lod: float, counter: EvalCounter | None = None):
    """Central-difference gradients, normalised (render.py:277-300).
    Returns (normals, ok)."""
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    k = len(pts)
    if k == 0:
        return np.zeros((0, 3)), np.zeros(0, dtype=bool)
    dev = _lib.device()
    cfg = resolve_config(fld, RenderConfig(), max(float(lod), 1.0), eps=eps)
    out = torch.empty((k, 3), dtype=torch.float64, device=dev)
    ok = torch.empty(k, dtype=torch.uint8, device=dev)
    c = _Counters()
    d_pts = torch.from_numpy(np.ascontiguousarray(pts)).to(dev)
    call("ng_normals", fld.svo.device.ref(), fld.device.ref(), ctypes.byref(cfg), ptr(d_pts), k, ptr(out), ptr(ok),
         c.ptr(), stream_ptr())
    ch = c.host()
    if ch[3]:
        raise OctfieldError("non-finite decoder input")
    if counter is not None:
        counter.add(ch)
    return out.cpu().numpy(), ok.cpu().numpy().astype(bool)


def shade(hit, nrm, config: RenderConfig) -> np.ndarray:
    """Lambert shading, 8-bit RGB (render.py:303-314)."""
    hit = np.asarray(hit, dtype=bool)
    nrm = np.asarray(nrm, dtype=np.float64)
    shape = hit.shape
    n = hit.size
    dev = _lib.device()
    c = _lib.NgRenderCfg()
    light = np.asarray(config.light_dir, dtype=np.float64)
    light = light / np.linalg.norm(light)
    for a in range(3):
        c.light[a] = float(light[a])
        c.albedo[a] = float(config.albedo[a])
        c.background[a] = float(config.background[a])
    c.ambient = float(config.ambient)
    out = torch.empty((max(n, 1), 3), dtype=torch.uint8, device=dev)
    if n:
        d_hit = torch.from_numpy(np.ascontiguousarray(hit.ravel()).astype(np.uint8)).to(dev)
        d_n = torch.from_numpy(np.ascontiguousarray(nrm.reshape(-1, 3))).to(dev)
        call("ng_shade", ptr(d_hit), ptr(d_n), n, ctypes.byref(c), ptr(out), stream_ptr())
    return out[:n].cpu().numpy().reshape(shape + (3,))


def write_ppm(path, image: np.ndarray) -> None:
    """Binary P6, 8-bit (render.py:317-324)."""
    if image.ndim != 3 or image.shape[2] != 3 or image.dtype != np.uint8:
        raise StructuralError("write_ppm expects (h, w, 3) uint8")
    h, w = image.shape[:2]
    with open(path, "wb") as fh:
        fh.write(f"P6\n{w} {h}\n255\n".encode("ascii"))
        fh.write(image.tobytes())


def normal_image(fb: FrameBuffer) -> np.ndarray:
    rgb = np.where(fb.hit[..., None], 0.5 * (fb.normal + 1.0), 0.0)
    return (np.clip(rgb, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)


def depth_image(fb: FrameBuffer, far: float) -> np.ndarray:
    g = np.where(fb.hit, 1.0 - np.nan_to_num(fb.t) / far, 0.0)
    g = (np.clip(g, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)
    return np.repeat(g[..., None], 3, axis=2)


# ------------------------------------------------------------------ frames

def resolve_lod(camera: Camera, fld: NeuralField, config: RenderConfig) -> float:
    """render.py:345-353."""
    if config.lod is not None:
        lod = float(config.lod)
        if lod > fld.max_level:
            raise ConfigError(f"lod {lod} above max level {fld.max_level}")
    elif config.lod_thresholds is not None:
        lod = select_lod(camera, fld.svo, config.lod_thresholds)
    else:
        lod = float(fld.max_level)
    return max(lod, 1.0)


_CAPTURE_LOCK = threading.Lock()


class _NativeGraph:
    """One frame's launches captured as a CUDA graph through the library
    (ng_graph_*): captured on a side stream in thread-local mode, replayed
    on the current stream. Unlike torch.cuda.graph, capturing does not
    synchronise the device or empty torch's device and pinned-host caches,
    so a streaming loop meeting a new launch key keeps its cached blocks
    (and its frame-buffer addresses, hence its graph keys)."""

    def __init__(self, launch, side: torch.cuda.Stream):
        side.wait_stream(torch.cuda.current_stream())
        h = ctypes.c_void_p()
        with _CAPTURE_LOCK:  # (one capture at a time per process keeps errors attributable)
            call("ng_graph_capture_begin", side.cuda_stream)
            try:
                launch(side.cuda_stream)
            except BaseException:
                # leave the stream out of capture mode before reporting
                _lib.lib().ng_graph_capture_end(ctypes.c_void_p(side.cuda_stream), ctypes.byref(h))
                if h.value:
                    _lib.lib().ng_graph_destroy(h)
                raise
            call("ng_graph_capture_end", side.cuda_stream, ctypes.byref(h))
        self.h = h.value

    def replay(self):
        call("ng_graph_launch", self.h, stream_ptr())

    def __del__(self):
        try:
            if self.h:
                _lib.lib().ng_graph_destroy(ctypes.c_void_p(self.h))
        except Exception:
            pass


def _graphs_enabled() -> bool:
    """NG_GRAPHS=0 launches every frame's kernels directly."""
    return os.environ.get("NG_GRAPHS", "1") != "0" and os.environ.get("NG_MARCH_PROFILE") != "1"


class FrameTensors:
    """One frame's device outputs in a single allocation. The C side gets
    raw pointers (no per-field tensor ops on the per-frame path); a field's
    tensor view is made on first access, `frame["color"]` etc."""

    # name: (byte offset per pixel, bytes per pixel, dtype, trailing shape)
    _LAYOUT = {"t": (0, 8, torch.float64, ()), "normal": (8, 24, torch.float64, (3,)),
               "iterations": (32, 4, torch.int32, ()), "evals": (36, 4, torch.int32, ()),
               "hit": (40, 1, torch.uint8, ()), "normal_ok": (41, 1, torch.uint8, ()),
               "color": (42, 3, torch.uint8, (3,))}
    BYTES_PER_PIXEL = 45

    def __init__(self, n: int, dev):
        self.n = n
        self.buf = torch.empty(self.BYTES_PER_PIXEL * n, dtype=torch.uint8, device=dev)
        self._views = {}

    def struct(self) -> _lib.NgFrame:
        b, n = self.buf.data_ptr(), self.n
        off = {k: b + v[0] * n for k, v in self._LAYOUT.items()}
        return _lib.NgFrame(off["hit"], off["t"], off["normal"], off["normal_ok"], off["iterations"], off["evals"],
                            off["color"])

    def __getitem__(self, name):
        v = self._views.get(name)
        if v is None:
            o, w, dt, tail = self._LAYOUT[name]
            n = self.n
            v = self.buf[o * n:(o + w) * n].view(dt).view((n,) + tail)
            self._views[name] = v
        return v

    def __contains__(self, name):
        return name in self._LAYOUT


class RenderSession:
    """Reusable device state for rendering frames of one size: workspace,
    frame buffers, statistics. `enqueue` launches a frame with no host sync;
    `finish` reads the statistics and applies the reference's per-frame
    checks. Capacities grow (and the frame reruns) on overflow."""

    def __init__(self, fld: NeuralField, width: int, height: int, n_rays: int | None = None):
        self.fld = fld
        self.width, self.height = width, height
        self.n = n_rays if n_rays is not None else width * height
        self.pair_cap = max(8 * self.n, 1 << 16)
        self.hit_cap = max(4 * self.n, 1 << 16)
        self.dev = _lib.device()
        self._alloc_ws()
        self.stats = torch.zeros(ctypes.sizeof(_lib.NgFrameStats) // 8, dtype=torch.int64, device=self.dev)
        self.stats_host = torch.zeros_like(self.stats, device="cpu").pin_memory()
        self.ev0 = torch.cuda.Event(enable_timing=True)
        self.ev1 = torch.cuda.Event(enable_timing=True)
        self.ev2 = torch.cuda.Event(enable_timing=True)
        self._graphs, self._graph_seen, self._graph_misses = {}, set(), 0
        self.graph_replays = 0
        self._cap_stream = None  # the stream frame graphs are captured on

    def _alloc_ws(self):
        nbytes = _lib.lib().ng_render_workspace_bytes(self.n, self.pair_cap, self.hit_cap)
        self.ws_buf = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        self.ws = _lib.NgWorkspace(ptr(self.ws_buf), nbytes, self.pair_cap, self.hit_cap, None, None)

    def new_frame(self) -> "FrameTensors":
        """Fresh per-pixel output buffers (every frame owns its own, as the
        reference returns fresh arrays)."""
        return FrameTensors(self.n, self.dev)

    @staticmethod
    def frame_struct(fr) -> _lib.NgFrame:
        if isinstance(fr, FrameTensors):
            return fr.struct()
        return _lib.NgFrame(ptr(fr["hit"]), ptr(fr["t"]), ptr(fr["normal"]), ptr(fr["normal_ok"]),
                            ptr(fr["iterations"]), ptr(fr["evals"]), ptr(fr["color"]))

    def enqueue(self, cfg: _lib.NgRenderCfg, frame: dict, camera=None, rays: torch.Tensor | None = None,
                timed: bool = False, do_normals: bool = True) -> None:
        """Launch one frame on the current stream. With `timed`, ev0 / ev1 /
        ev2 bracket traversal+march and normals (ev1 is recorded by the C side).
        `camera` may be a list of cameras (or camera structs) of one size:
        a batch (ng_render_batch), frame f in pixels [f n, (f + 1) n) of
        `frame` (n = width * height)."""
        fs = self.frame_struct(frame)
        fstruct = prepare_presum(self.fld, cfg)
        graphed = camera is not None and _graphs_enabled() and self._graph_misses < 16
        if timed and not graphed:
            self.ev1.record()  # materialise the handle; re-recorded mid-frame
            self.ws.ev_trace_done = self.ev1.cuda_event
            self.ev0.record()
        else:
            self.ws.ev_trace_done = None
            if timed:
                self.ev0.record()
        if camera is not None:
            tree, field = self.fld.svo.device.ref(), ctypes.byref(fstruct)
            cs = camera_structs(camera)

            def launch(stream=None):
                call("ng_render_batch", tree, field, ctypes.byref(cfg), cs, len(cs), ctypes.byref(fs),
                     ctypes.byref(self.ws), ptr(self.stats), stream if stream is not None else stream_ptr())
            if graphed:
                # the frame's launches as one CUDA graph, replayed while every
                # argument is unchanged (render() reusing a freed frame buffer
                # gets the same address back from the caching allocator);
                # timed graphed frames are timed as a whole (ev0 -> ev1), the
                # normals being evaluated inside the march
                key = (bytes(self.fld.svo.device.struct), bytes(fstruct), bytes(cfg), bytes(cs),
                       bytes(fs), bytes(self.ws))
                g = self._graphs.get(key)
                if g is None and key not in self._graph_seen:
                    # first sight: launch directly (lazy one-off set-up stays
                    # outside any capture); captured on the next occurrence
                    self._graph_seen.add(key)
                    self._graph_misses += 1
                    launch()
                else:
                    if g is None:  # a few graphs: consecutive frames alternate buffers
                        # (render_frames keeps three frames alive: their
                        # buffers cycle through a handful of address sets)
                        if len(self._graphs) >= 16:
                            self._graphs.pop(next(iter(self._graphs)))
                        if self._cap_stream is None:
                            self._cap_stream = torch.cuda.Stream(device=self.dev)
                        g = _NativeGraph(launch, self._cap_stream)
                        self._graphs[key] = g
                    self._graph_misses = 0
                    self.graph_replays += 1
                    g.replay()
                if timed:
                    self.ev1.record()
            else:
                launch()
        else:
            call("ng_render_rays", self.fld.svo.device.ref(), ctypes.byref(fstruct), ctypes.byref(cfg), ptr(rays),
                 self.n, ctypes.byref(fs), ctypes.byref(self.ws), ptr(self.stats), int(do_normals), stream_ptr())
        if timed:
            self.ev2.record()
        self.ws.ev_trace_done = None

    def read_stats(self) -> _lib.NgFrameStats:
        self.stats_host.copy_(self.stats, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        raw = self.stats_host.numpy().tobytes()
        return _lib.NgFrameStats.from_buffer_copy(raw[:ctypes.sizeof(_lib.NgFrameStats)])

    def final_list(self, level: int, cells: bool = False):
        """The last frame's final (ray, voxel, t_enter, t_exit) list as the
        render path's traversal left it in the workspace, put in the
        reference's order (ray_trace_octree's last list, traversal.py:207-247:
        by ray, each ray's voxels front to back). Ray ids are local to this
        session's rays (a band camera's rows in band order). With `cells`,
        also the packed cell (x | y << 10 | z << 20) each entry carries on the
        tile path. Read after a frame without shadow rays (the shadow pass
        reuses the lists)."""
        off = (ctypes.c_int64 * 4)()
        _lib.check(_lib.lib().ng_render_workspace_offsets(self.n, self.pair_cap, self.hit_cap, off, 4),
                   "ng_render_workspace_offsets")
        torch.cuda.current_stream().synchronize()
        b = self.ws_buf
        s = b[off[1]:off[1] + 8 * self.n].view(torch.int64).cpu().numpy()
        e = b[off[2]:off[2] + 8 * self.n].view(torch.int64).cpu().numpy()
        lens = e - s
        total = int(lens.sum())
        used = int(e.max(initial=0))
        raw = b[off[0]:off[0] + _lib.HIT_PAIR_BYTES * used].cpu().numpy()
        rec = raw.view(np.dtype([("ray", "<i4"), ("voxel", "<i4"), ("t_enter", "<f8"), ("t_exit", "<f8")]))
        rays = np.repeat(np.arange(self.n, dtype=np.int64), lens)
        first = np.repeat(s - np.concatenate(([0], np.cumsum(lens)[:-1])), lens)
        idx = first + np.arange(total, dtype=np.int64)
        out = RayVoxelPairList(level, rays, rec["voxel"][idx].astype(np.int64), rec["t_enter"][idx].copy(),
                               rec["t_exit"][idx].copy())
        if cells:
            return out, rec["ray"][idx].astype(np.int64)
        return out

    def grow(self, st: _lib.NgFrameStats, n_levels: int) -> bool:
        """Grow capacities after an overflow; True when a rerun is needed."""
        if not st.overflow:
            return False
        need_pairs = max(st.pairs[t] for t in range(1, n_levels))
        self.pair_cap = max(self.pair_cap, int(need_pairs) + 4096, int(st.pair_need))
        self.hit_cap = max(self.hit_cap, int(st.pairs[n_levels]) + 4096)
        self._alloc_ws()
        return True


_SESSIONS = threading.local()


def _session(fld: NeuralField, width: int, height: int, frames: int = 1) -> RenderSession:
    """render()'s reusable frame state, per calling thread, device and
    stream (concurrent callers never share a workspace; SURVEY.md 8b
    Threading); `frames` > 1: room for a batch of that many frames."""
    cache = getattr(_SESSIONS, "d", None)
    if cache is None:
        cache = _SESSIONS.d = {}
    key = (id(fld), width, height, frames, torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream)
    s = cache.get(key)
    if s is None or s.fld is not fld:
        if len(cache) > 8:
            cache.clear()
        s = RenderSession(fld, width, height, n_rays=width * height * frames)
        cache[key] = s
    return s


def camera_structs(cameras):
    """ng_camera array of one camera or a batch (Camera objects or structs)."""
    if isinstance(cameras, (Camera, _lib.NgCamera)):
        cameras = [cameras]
    cams = [c.struct() if isinstance(c, Camera) else c for c in cameras]
    if not 1 <= len(cams) <= _lib.MAX_BATCH:
        raise ConfigError(f"a batch holds 1..{_lib.MAX_BATCH} cameras, got {len(cams)}")
    arr = (_lib.NgCamera * len(cams))()
    for i, c in enumerate(cams):
        arr[i] = c
    return arr


class _FrameSlice:
    """Frame f of a batch's stacked device outputs (a FrameBuffer's `dev`)."""

    def __init__(self, frame: "FrameTensors", f: int, n: int):
        self.frame, self.lo, self.hi = frame, f * n, (f + 1) * n

    def __getitem__(self, name):
        return self.frame[name][self.lo:self.hi]


def _batch_cfg(cameras, fld: NeuralField, config: RenderConfig):
    """The batch's resolved configuration: every camera of one size, and one
    detail level (a camera-dependent LOD must resolve alike for all)."""
    w, h = cameras[0].width, cameras[0].height
    if any(c.width != w or c.height != h for c in cameras):
        raise ConfigError("a batch's cameras must share one image size")
    lods = [resolve_lod(c, fld, config) for c in cameras]
    if any(l != lods[0] for l in lods):
        raise ConfigError("a batch's cameras resolve to different detail levels: render them separately")
    return lods[0], resolve_config(fld, config, lods[0])


def render_batch(cameras, fld: NeuralField, config: RenderConfig):
    """Render up to MAX_BATCH cameras of one size in one launch sequence
    (ng_render_batch): one traversal and one march over every frame's rays,
    so the frames' longest rays overlap each other's work instead of each
    frame ending on its own. Returns (list of FrameBuffer, FrameReport);
    each frame equals `render(camera, ...)`'s, the report covers the batch
    (its `visible`, `evals` and times are the batch's totals)."""
    cameras = list(cameras)
    if not 1 <= len(cameras) <= _lib.MAX_BATCH:
        raise ConfigError(f"a batch holds 1..{_lib.MAX_BATCH} cameras, got {len(cameras)}")
    lod, cfg = _batch_cfg(cameras, fld, config)
    k = len(cameras)
    w, h = cameras[0].width, cameras[0].height
    sess = _session(fld, w, h, k)
    n_levels = cfg.trace_level + fld.svo.device.n_virtual
    while True:
        frame = sess.new_frame()
        sess.enqueue(cfg, frame, camera=cameras, timed=True)
        color_h = torch.empty(frame["color"].shape, dtype=torch.uint8, pin_memory=True)
        color_h.copy_(frame["color"], non_blocking=True)
        st = sess.read_stats()
        if not sess.grow(st, n_levels):
            break
    if st.counters.nonfinite_inputs:
        raise OctfieldError("non-finite decoder input")
    if st.counters.evals_missing_level != 0:
        raise OctfieldError("internal: decoder ran outside the queried level's voxels")
    n = w * h
    fbs = [FrameBuffer(w, h, _FrameSlice(frame, f, n), camera=c, prefetched={"color": color_h[f * n:(f + 1) * n]})
           for f, c in enumerate(cameras)]
    report = FrameReport(ms_trace=float(sess.ev0.elapsed_time(sess.ev1)), ms_normals=float(sess.ev1.elapsed_time(sess.ev2)),
                         evals=int(st.counters.decoder_evals), visible=int(st.visible), lod=lod,
                         shadowed=int(st.shadowed))
    return fbs, report


def render(camera: Camera, fld: NeuralField, config: RenderConfig):
    """Trace a frame (render.py:342-448). Returns (FrameBuffer, FrameReport);
    the report times traversal + march and the normals separately with CUDA
    events, matching the benchmark scope."""
    lod = resolve_lod(camera, fld, config)
    cfg = resolve_config(fld, config, lod)
    sess = _session(fld, camera.width, camera.height)
    n_levels = cfg.trace_level + fld.svo.device.n_virtual  # index of the final hit count
    while True:
        frame = sess.new_frame()
        sess.enqueue(cfg, frame, camera=camera, timed=True)
        # the colour image rides the same stream synchronisation as the statistics
        color_h = torch.empty(frame["color"].shape, dtype=torch.uint8, pin_memory=True)
        color_h.copy_(frame["color"], non_blocking=True)
        st = sess.read_stats()
        if not sess.grow(st, n_levels):
            break
    if st.counters.nonfinite_inputs:
        raise OctfieldError("non-finite decoder input")
    if st.counters.evals_missing_level != 0:
        raise OctfieldError("internal: decoder ran outside the queried level's voxels")
    ms_trace = sess.ev0.elapsed_time(sess.ev1)
    ms_normals = sess.ev1.elapsed_time(sess.ev2)
    fb = FrameBuffer(camera.width, camera.height, frame, camera=camera, prefetched={"color": color_h})
    report = FrameReport(ms_trace=float(ms_trace), ms_normals=float(ms_normals),
                         evals=int(st.counters.decoder_evals), visible=int(st.visible), lod=lod,
                         shadowed=int(st.shadowed))
    return fb, report


def _chunks(cameras, fld: NeuralField, config: RenderConfig, batch: int):
    """Consecutive cameras grouped into batches of up to `batch` that share
    an image size and a resolved configuration."""
    cur, key0 = [], None
    for camera in cameras:
        lod = resolve_lod(camera, fld, config)
        cfg = resolve_config(fld, config, lod)
        key = (camera.width, camera.height, bytes(cfg))
        if cur and (key != key0 or len(cur) == batch):
            yield cur
            cur = []
        if not cur:
            key0 = key
        cur.append((camera, lod, cfg))
    if cur:
        yield cur


def render_frames(cameras, fld: NeuralField, config: RenderConfig, batch: int = 1):
    """Render a sequence of cameras; yields (FrameBuffer, FrameReport) per
    camera, in order, exactly as `render` returns them. Frame i + 1 is
    launched before frame i's colour image and statistics are read back
    (double-buffered readback): each frame's device-to-host copies and host
    work overlap the next frame's kernels, the way a real-time loop
    consumes frames. With `batch` > 1, up to `batch` consecutive cameras of
    one size and detail level go in one launch sequence (`render_batch`),
    and each of their reports covers that batch. A batch whose lists
    overflowed is grown and re-rendered before it is yielded.
    `report.ms_trace` is the launch's device time (the normals run inside
    the march)."""
    if not 1 <= batch <= _lib.MAX_BATCH:
        raise ConfigError(f"batch must be 1..{_lib.MAX_BATCH}, got {batch}")
    pending = None
    stats_host = {}
    k = 0
    copy = torch.cuda.Stream()  # the colour readback runs beside the next frame's kernels
    for chunk in _chunks(cameras, fld, config, batch):
        cams = [c for c, _, _ in chunk]
        lod, cfg = chunk[0][1], chunk[0][2]
        w, h = cams[0].width, cams[0].height
        sess = _session(fld, w, h, batch)
        frame = sess.new_frame()
        ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev_a.record()
        sess.enqueue(cfg, frame, camera=cams if len(cams) > 1 else cams[0])
        ev_b.record()
        # the statistics (one small buffer every frame writes) are copied on
        # the frame's stream; the colour images on the copy stream, so their
        # transfer overlaps the next launch instead of queueing before it
        key = (id(sess), k % 2)
        st_h = stats_host.get(key)
        if st_h is None:
            st_h = stats_host[key] = torch.zeros_like(sess.stats, device="cpu").pin_memory()
        st_h.copy_(sess.stats, non_blocking=True)
        done = torch.cuda.Event()
        done.record()
        color = frame["color"][:len(cams) * w * h]
        color_h = torch.empty(color.shape, dtype=torch.uint8, pin_memory=True)
        copy.wait_event(ev_b)
        with torch.cuda.stream(copy):
            color_h.copy_(color, non_blocking=True)
        color.record_stream(copy)  # (the caching allocator keeps the buffer until the copy ran)
        done_copy = torch.cuda.Event()
        done_copy.record(copy)
        done = (done, done_copy)
        if pending is not None:
            yield from _finish_frames(*pending)
        pending = (cams, fld, config, lod, sess, frame, color_h, st_h, done, ev_a, ev_b)
        k += 1
    if pending is not None:
        yield from _finish_frames(*pending)


def _finish_frames(cams, fld, config, lod, sess, frame, color_h, st_h, done, ev_a, ev_b):
    for ev in done:
        ev.synchronize()
    raw = st_h.numpy().tobytes()
    st = _lib.NgFrameStats.from_buffer_copy(raw[:ctypes.sizeof(_lib.NgFrameStats)])
    n_levels = resolve_config(fld, config, lod).trace_level + fld.svo.device.n_virtual
    if st.overflow:  # grow, then this launch again (synchronously)
        sess.grow(st, n_levels)
        if len(cams) == 1:
            yield render(cams[0], fld, config)
            return
        fbs, rep = render_batch(cams, fld, config)
        for fb in fbs:
            yield fb, rep
        return
    if st.counters.nonfinite_inputs:
        raise OctfieldError("non-finite decoder input")
    if st.counters.evals_missing_level != 0:
        raise OctfieldError("internal: decoder ran outside the queried level's voxels")
    report = FrameReport(ms_trace=float(ev_a.elapsed_time(ev_b)), ms_normals=0.0,
                         evals=int(st.counters.decoder_evals), visible=int(st.visible), lod=lod,
                         shadowed=int(st.shadowed))
    w, h = cams[0].width, cams[0].height
    n = w * h
    for f, camera in enumerate(cams):
        dev = frame if len(cams) == 1 else _FrameSlice(frame, f, n)
        fb = FrameBuffer(w, h, dev, camera=camera, prefetched={"color": color_h[f * n:(f + 1) * n]})
        yield fb, report


def trace_rays(fld: NeuralField, rays: RayBundle, lod: float, config: RenderConfig | None = None):
    """(hit, t_hit) for arbitrary rays with the renderer's rules; the
    device version of metrics.trace_field_rays (metrics.py:135-142)."""
    config = config or RenderConfig()
    lod = max(float(lod), 1.0)
    cfg = resolve_config(fld, config, lod)
    n = rays.count
    if n == 0:
        return np.zeros(0, dtype=bool), np.zeros(0)
    sess = RenderSession(fld, n, 1, n_rays=n)
    d_rays = device_rays(rays)
    n_levels = cfg.trace_level + fld.svo.device.n_virtual  # index of the final hit count
    while True:
        frame = sess.new_frame()
        sess.enqueue(cfg, frame, rays=d_rays, do_normals=False)
        st = sess.read_stats()
        if not sess.grow(st, n_levels):
            break
    if st.counters.nonfinite_inputs:
        raise OctfieldError("non-finite decoder input")
    return frame["hit"].cpu().numpy().astype(bool), frame["t"].cpu().numpy()
