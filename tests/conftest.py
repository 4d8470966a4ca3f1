import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(autouse=True)
def _drain_gpu(request):
    """After every GPU test, wait for the device: work a test left queued
    (a side stream, an unsynchronised launch) is charged to that test, not
    to whichever test next shares the GPU."""
    yield
    if request.node.get_closest_marker("gpu") is None:
        return
    import torch
    if torch.cuda.is_available() and torch.cuda.is_initialized():
        torch.cuda.synchronize()


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
        return cache[name]
    return load


def oracle_tree_from_golden(g, prefix):
    """Rebuild an OracleOctree from the fixture arrays written by
    tests/golden/make_golden.py."""
    from oracle.nglod_oracle import OracleOctree
    L = int(g[prefix + "max_level"])
    nv = int(g[prefix + "n_virtual"])
    return OracleOctree(
        r0=int(g[prefix + "r0"]), max_level=L,
        codes=[g[f"{prefix}codes{lv}"] for lv in range(L + 1)],
        parents=[g[f"{prefix}parents{lv}"] for lv in range(L + 1)],
        corners=[None] + [g[f"{prefix}corners{lv}"] for lv in range(1, L + 1)],
        corner_offsets=g[prefix + "corner_offsets"],
        corner_count=int(g[prefix + "corner_count"]),
        region_lo=g[prefix + "region_lo"], region_hi=g[prefix + "region_hi"],
        virtual_codes=[g[f"{prefix}vcodes{i}"] for i in range(nv)],
    )


@pytest.fixture(scope="session")
def reference():
    """The live reference package, only where /root/reference exists."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference sources not present on this machine")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import octfield
    import octfield.render  # noqa: F401
    return octfield
