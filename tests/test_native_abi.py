"""CPU checks of the C-ABI library and the host layer (no compute calls)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "nglod_b200.h")
LIB = os.path.join(ROOT, "paper_2101_10994_b200", "libnglod_b200.so")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ng_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB)
    missing = [s for s in _declared() if not hasattr(lib, s)]
    assert not missing, f"declared but not exported: {missing}"
    assert lib.ng_abi_version() == 1


def test_binding_covers_header():
    from paper_2101_10994_b200 import _lib
    assert sorted(_lib.EXPORTED) == _declared()


def test_struct_sizes_match_header_layout():
    from paper_2101_10994_b200 import _lib
    assert ctypes.sizeof(_lib.NgOctree) == 16 + 16 * 8 + 6 * 16 * 8 + 7 * 8
    assert ctypes.sizeof(_lib.NgField) == 40 + 8 + 8 + 8 + 4 + 4  # + presum table pointer, offset, corners, level, mask
    assert ctypes.sizeof(_lib.NgQueryArgs) == 24
    assert ctypes.sizeof(_lib.NgCamera) == 12 * 8 + 2 * 8 + 6 * 4
    assert ctypes.sizeof(_lib.NgFrameStats) == (17 + 2 + 4 + 1 + 17 + 1 + 1) * 8
    assert _lib.RAY_BYTES == 80 and _lib.HIT_PAIR_BYTES == 24


def test_host_validation_before_device():
    """Errors the reference raises on bad input are raised by the host
    layer before any device work (octree.py:163-169, render.py:52-114)."""
    import paper_2101_10994_b200 as ng
    with pytest.raises(ng.StructuralError):
        ng.build_octree(None, 0, np.zeros((1, 3)))
    with pytest.raises(ng.StructuralError):
        ng.build_octree(None, 1, np.zeros((1, 3)), r0=3)
    with pytest.raises(ng.StructuralError):
        ng.morton_encode(np.array([[2**21, 0, 0]]))
    with pytest.raises(ng.ConfigError):
        ng.RenderConfig(delta=0.0)
    with pytest.raises(ng.ConfigError):
        ng.RenderConfig(max_iters=0)
    with pytest.raises(ng.ConfigError):
        ng.Camera((0, 0, 4), (0, 0, 0), (0, 1, 0), 0.0, 8, 8)
    with pytest.raises(ng.ConfigError):
        ng.Camera((0, 0, 4), (0, 0, 0), (0, 0, 1), 30.0, 8, 8)
    with pytest.raises(ng.StructuralError):
        ng.RayBundle(np.zeros((2, 3)), np.array([[1.0, 1.0, 0.0], [0.0, 0.0, 1.0]]))
    # frame batches: 1..NG_MAX_BATCH cameras per launch, checked before the field is touched
    cam = ng.Camera((0, 0, 4), (0, 0, 0), (0, 1, 0), 30.0, 8, 8)
    import re
    from paper_2101_10994_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "nglod_b200.h")).read()
    assert int(re.search(r"#define NG_MAX_BATCH (\d+)", hdr).group(1)) == _lib.MAX_BATCH
    with pytest.raises(ng.ConfigError):
        ng.render_batch([cam] * (_lib.MAX_BATCH + 1), None, ng.RenderConfig())
    with pytest.raises(ng.ConfigError):
        ng.render_batch([], None, ng.RenderConfig())
    with pytest.raises(ng.ConfigError):
        next(ng.render_frames([cam], None, ng.RenderConfig(), batch=0))
    from paper_2101_10994_b200.render import camera_structs
    assert len(camera_structs([cam] * _lib.MAX_BATCH)) == _lib.MAX_BATCH
    with pytest.raises(ng.ConfigError):
        camera_structs([cam] * (_lib.MAX_BATCH + 1))


def test_no_device_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    import paper_2101_10994_b200 as ng
    from paper_2101_10994_b200 import _lib
    with pytest.raises(_lib.NativeUnavailable):
        ng.build_octree(None, 1, np.array([[0.5, 0.5, 0.5]]), corner_test=False)


def test_decoder_packing_layout():
    from paper_2101_10994_b200 import field
    rng = np.random.default_rng(0)
    d = field.Decoder(rng.standard_normal((16, 11)).astype(np.float32), rng.standard_normal(16).astype(np.float32),
                      rng.standard_normal((1, 16)).astype(np.float32), np.array([0.5], np.float32))
    buf = field.pack_decoders([d], 8)
    stride = field.decoder_stride(16)
    assert buf.shape == (1, stride) and stride % 4 == 0
    blk = buf[0, :16 * 36].reshape(16, 36)
    np.testing.assert_array_equal(blk[:, :11], d.W1)
    np.testing.assert_array_equal(blk[:, 11:35], 0.0)
    np.testing.assert_array_equal(blk[:, 35], d.b1)
    np.testing.assert_array_equal(buf[0, 16 * 36:16 * 36 + 16], d.W2[0])
    assert buf[0, 16 * 36 + 16] == np.float32(0.5)
