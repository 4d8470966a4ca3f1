"""ctypes binding of the C ABI in include/nglod_b200.h.

The shared library `libnglod_b200.so` is built in-tree for sm_100a
(`__graft_entry__.build()` / `make -C paper_2101_10994_b200/csrc`). There is
no fallback: importing a function that needs the device raises
`NativeUnavailable` when the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from .errors import ConfigError, OctfieldError, StructuralError

HERE = os.path.dirname(os.path.abspath(__file__))
# NG_LIB_VARIANT=name loads variants/libnglod_<name>.so (tools/build_variant.sh:
# the same sources with different compile-time knobs, for A/B timing)
LIB_PATH = (os.path.join(HERE, "variants", f"libnglod_{os.environ['NG_LIB_VARIANT']}.so")
            if os.environ.get("NG_LIB_VARIANT") else os.path.join(HERE, "libnglod_b200.so"))

NG_OK = 0
NG_ERR_STRUCTURAL = 1
NG_ERR_CONFIG = 2
NG_ERR_CAPACITY = 3
NG_ERR_CUDA = 4
NG_ERR_OCTFIELD = 5

MAX_TLEVELS = 16
MAX_BATCH = 16  # NG_MAX_BATCH: cameras per ng_render_batch launch
FEAT_PAD = 32
W1_STRIDE = 36


class NativeUnavailable(RuntimeError):
    """The CUDA library or device is missing; there is no CPU fallback."""


class CapacityError(OctfieldError):
    """Internal: a device buffer was too small (callers grow and retry)."""


# ----------------------------------------------------------------- structs

P = C.c_void_p


class NgOctree(C.Structure):
    _fields_ = [
        ("r0", C.c_int32), ("max_level", C.c_int32), ("n_virtual", C.c_int32), ("n_tlevels", C.c_int32),
        ("count", C.c_int64 * MAX_TLEVELS),
        ("codes", P * MAX_TLEVELS),
        ("child_start", P * MAX_TLEVELS),
        ("child_mask", P * MAX_TLEVELS),
        ("bitmap", P * MAX_TLEVELS),
        ("rank", P * MAX_TLEVELS),
        ("corners", P * MAX_TLEVELS),
        ("region_lo", C.c_double * 3),
        ("region_hi", C.c_double * 3),
        ("half_diag_finest", C.c_double),
    ]


class NgField(C.Structure):
    _fields_ = [
        ("Z", P), ("decoders", P), ("m", C.c_int32), ("h", C.c_int32),
        ("n_decoders", C.c_int32), ("dec_stride", C.c_int32), ("corner_count", C.c_int64),
        ("presum", P), ("presum_offset", C.c_int64), ("presum_corners", C.c_int64), ("presum_level", C.c_int32),
        ("presum_mask", C.c_int32),
    ]


class NgCounters(C.Structure):
    _fields_ = [("decoder_evals", C.c_int64), ("evals_missing_level", C.c_int64),
                ("empty_fallbacks", C.c_int64), ("nonfinite_inputs", C.c_int64)]


class NgQueryArgs(C.Structure):
    _fields_ = [("out_levels", C.c_int32), ("inside_level", C.c_int32), ("blend_base", C.c_int32),
                ("pad", C.c_int32), ("blend_alpha", C.c_double)]


class NgCamera(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("fwd", C.c_double * 3), ("right", C.c_double * 3),
                ("up", C.c_double * 3), ("tan_half", C.c_double), ("aspect", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("band_rows", C.c_int32),
                ("band_stride", C.c_int32), ("band_offset", C.c_int32), ("local_rows", C.c_int32)]


class NgRenderCfg(C.Structure):
    _fields_ = [("delta", C.c_double), ("far_plane", C.c_double), ("skip_eps", C.c_double),
                ("osc_tol", C.c_double), ("lod", C.c_double), ("normal_eps", C.c_double),
                ("light", C.c_double * 3), ("albedo", C.c_double * 3), ("ambient", C.c_double),
                ("background", C.c_double * 3), ("max_iters", C.c_int32), ("trace_level", C.c_int32),
                ("shadow_offset", C.c_double), ("shadows", C.c_int32), ("pad", C.c_int32)]


class NgFrame(C.Structure):
    _fields_ = [("hit", P), ("t", P), ("normal", P), ("normal_ok", P), ("iterations", P),
                ("evals", P), ("color", P)]


class NgWorkspace(C.Structure):
    _fields_ = [("base", P), ("bytes", C.c_size_t), ("pair_capacity", C.c_int64),
                ("hit_capacity", C.c_int64), ("ev_trace_done", P), ("ev_march_begin", P)]


class NgFrameStats(C.Structure):
    _fields_ = [("pairs", C.c_int64 * (MAX_TLEVELS + 1)), ("visible", C.c_int64),
                ("active_rays", C.c_int64), ("counters", NgCounters), ("overflow", C.c_int64),
                ("shadow_pairs", C.c_int64 * (MAX_TLEVELS + 1)), ("shadowed", C.c_int64),
                ("pair_need", C.c_int64)]


class NgTrainParams(C.Structure):
    _fields_ = [("Z", P), ("Zm", P), ("Zv", P), ("Zlast", P), ("dec", P), ("decm", P), ("decv", P), ("m", C.c_int32),
                ("h", C.c_int32), ("n_decoders", C.c_int32), ("dec_stride", C.c_int32),
                ("corner_count", C.c_int64)]


class NgTrainStep(C.Structure):
    _fields_ = [("active_mask", C.c_int32), ("update_decoders", C.c_int32), ("mode", C.c_int32),
                ("pad", C.c_int32), ("denom", C.c_double), ("lr", C.c_double), ("step", C.c_int64),
                ("adam_c", P), ("batch_index", C.c_int64)]


RAY_BYTES = 80
PAIR_BYTES = 8
HIT_PAIR_BYTES = 24

# ----------------------------------------------------------------- loading

_SIGS = {
    "ng_abi_version": (C.c_int, []),
    "ng_last_error": (C.c_char_p, []),
    "ng_sm_count": (C.c_int, [C.c_int]),
    "ng_morton_encode": (C.c_int, [P, C.c_int64, P, P]),
    "ng_morton_decode": (C.c_int, [P, C.c_int64, P, P]),
    "ng_locate": (C.c_int, [P, P, C.c_int64, C.c_int32, P, P]),
    "ng_ray_aabb": (C.c_int, [P, P, P, P, C.c_int64, P, P, P, P]),
    "ng_build_mark_samples": (C.c_int, [P, C.c_int64, C.c_int32, P, P]),
    "ng_build_mark_lattice": (C.c_int, [P, C.c_int32, C.c_double, P, P]),
    "ng_sdf_lattice": (C.c_int, [C.c_int32, P, C.c_int32, C.c_int32, P, P]),
    "ng_sdf_eval": (C.c_int, [C.c_int32, P, C.c_int32, P, C.c_int64, P, P]),
    "ng_bitmap_parent": (C.c_int, [P, C.c_int64, P, C.c_int64, P]),
    "ng_bitmap_rank": (C.c_int, [P, C.c_int64, P, P, P, C.c_size_t, P]),
    "ng_bitmap_extract": (C.c_int, [P, P, C.c_int64, P, P]),
    "ng_level_parents": (C.c_int, [P, C.c_int64, P, P, P, P]),
    "ng_level_children": (C.c_int, [P, C.c_int64, P, P, P, P, P]),
    "ng_corner_mark": (C.c_int, [P, C.c_int64, P, P]),
    "ng_corner_table": (C.c_int, [P, C.c_int64, P, P, C.c_int32, P, P]),
    "ng_cell_extent": (C.c_int, [P, C.c_int64, P, P]),
    "ng_scan_scratch_bytes": (C.c_size_t, [C.c_int64]),
    "ng_exclusive_sum_i64": (C.c_int, [P, C.c_int64, P, P, C.c_size_t, P]),
    "ng_query": (C.c_int, [P, P, P, P, C.c_int64, P, P, P]),
    "ng_interp": (C.c_int, [P, P, P, C.c_int64, C.c_int32, C.c_int32, P, P, P]),
    "ng_empty_value": (C.c_int, [P, P, C.c_int64, P, P]),
    "ng_interp64": (C.c_int, [P, P, C.c_int32, P, C.c_int64, C.c_int32, C.c_int32, P, P, P]),
    "ng_decode64": (C.c_int, [P, C.c_int32, C.c_int32, P, P, C.c_int64, P, P, P]),
    "ng_query64": (C.c_int, [P, P, C.c_int32, P, C.c_int32, C.c_int32, C.c_int32, P, P, C.c_int64, P, P, P]),
    "ng_decode": (C.c_int, [P, C.c_int32, C.c_int32, P, P, C.c_int64, P, P, P]),
    "ng_rays_from_arrays": (C.c_int, [P, P, C.c_int64, P, P]),
    "ng_level_scratch_bytes": (C.c_size_t, [C.c_int64]),
    "ng_traverse_level": (C.c_int, [P, P, C.c_int32, C.c_int32, P, P, C.c_int64, P, P, P, C.c_int64,
                                    P, C.c_size_t, P]),
    "ng_decide": (C.c_int, [P, P, C.c_int32, C.c_int32, P, C.c_int64, P, P]),
    "ng_subdivide": (C.c_int, [P, P, C.c_int32, P, C.c_int64, P, P, P, P]),
    "ng_compactify": (C.c_int, [P, C.c_int64, P, P, P, P]),
    "ng_segments": (C.c_int, [P, P, C.c_int64, C.c_int64, P, P, P]),
    "ng_camera_rays": (C.c_int, [P, P, P]),
    "ng_render_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int64, C.c_int64]),
    "ng_render_workspace_offsets": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, P, C.c_int32]),
    "ng_sphere_trace": (C.c_int, [P, P, P, P, C.c_int64, P, P, P, P, P, P, P, P, P, P]),
    "ng_normals": (C.c_int, [P, P, P, P, C.c_int64, P, P, P, P]),
    "ng_shade": (C.c_int, [P, P, C.c_int64, P, P, P]),
    "ng_render_frame": (C.c_int, [P, P, P, P, P, P, P, P]),
    "ng_render_batch": (C.c_int, [P, P, P, P, C.c_int32, P, P, P, P]),
    "ng_graph_capture_begin": (C.c_int, [P]),
    "ng_graph_capture_end": (C.c_int, [P, C.POINTER(C.c_void_p)]),
    "ng_graph_launch": (C.c_int, [P, P]),
    "ng_graph_destroy": (C.c_int, [P]),
    "ng_render_rays": (C.c_int, [P, P, P, P, C.c_int64, P, P, P, C.c_int32, P]),
    "ng_hit_points": (C.c_int, [P, P, P, C.c_int64, P, P]),
    "ng_march_profile": (C.c_int, [P, C.c_int]),
    "ng_train_workspace_bytes": (C.c_size_t, [P, C.c_int64, C.c_int32, C.c_int32, C.c_int64, C.c_int32]),
    "ng_train_batch": (C.c_int, [P, P, P, P, P, P, C.c_int64, C.c_int64, P, C.c_size_t, P, P, P, P, P, P, P]),
    "ng_train_epoch": (C.c_int, [P, P, P, P, C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_double,
                                 C.c_int64, P, C.c_int32, P, C.c_size_t, P, P, P]),
    "ng_train_flush": (C.c_int, [P, C.c_int64, P, C.c_double, P]),
    "ng_train_profile": (C.c_int, [P]),
    "ng_train_export": (C.c_int, [P, P, C.c_int32, P, C.c_int64, P, C.c_size_t, P, P, P, P, P, P]),
    "ng_field_presum": (C.c_int, [P, P, C.c_int32, C.c_int32, C.c_int64, C.c_int64, P, P, P]),
    "ng_trace_sdf": (C.c_int, [C.c_int32, P, C.c_int32, P, P, C.c_int64, C.c_double, C.c_double, C.c_int32, P, P,
                               P]),
    "ng_nearest_voxel": (C.c_int, [P, C.c_int32, P, C.c_int64, P, P, P]),
    "ng_nn_dist": (C.c_int, [P, C.c_int64, P, C.c_int64, P, P]),
    "ng_surface_trace": (C.c_int, [C.c_int32, P, C.c_int32, P, P, C.c_int64, C.c_double, C.c_double, C.c_int32,
                                   C.c_int32, P, P]),
    "ng_adam_step": (C.c_int, [P, P, P, P, C.c_int64, C.c_double, C.c_double, C.c_double, P, P]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load_library(path: str = LIB_PATH):
    """Load the shared library and declare every entry point's signature."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    """The library, after checking a CUDA device is present."""
    L = load_library()
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the nglod_b200 path has no CPU fallback")
    return L


def check(status: int, what: str = "") -> None:
    if status == NG_OK:
        return
    msg = (_lib.ng_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == NG_ERR_STRUCTURAL:
        raise StructuralError(text)
    if status == NG_ERR_CONFIG:
        raise ConfigError(text)
    if status == NG_ERR_CAPACITY:
        raise CapacityError(text)
    if status == NG_ERR_OCTFIELD:
        raise OctfieldError(text)
    raise RuntimeError(f"CUDA failure in {text}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def device() -> torch.device:
    """The current CUDA device; raises NativeUnavailable without one (or
    without the library) -- there is no host fallback."""
    lib()
    return torch.device("cuda", torch.cuda.current_device())
