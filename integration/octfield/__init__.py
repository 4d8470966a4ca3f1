"""`octfield` with its hot path swapped for the B200 implementation.

Put `integration/` ahead of the reference on sys.path and `import octfield`
gives the reference's own package surface (its __init__.py is executed
here, unchanged) in which the hot-path modules ARE this repository's:

    octfield.errors, octree, field, traversal, render, trainer, modelio,
    metrics  ->  paper_2101_10994_b200.<same name>

while the modules outside the hot path (geometry: analytic/mesh oracles and
the CSG scene parser; sampling's mesh samplers; the cli) are the
reference's source files, executed as `octfield.<name>` so their relative
imports (`from .errors import ...`, `from .render import ...`) resolve to
the swapped modules. Exceptions are therefore one set of classes.

The reference source is found in $OCTFIELD_REF_SRC, else
baseline/_ref/octfield (pip install --target baseline/_ref), else
/root/reference/pkg/src/octfield. tests/test_gpu_reference_suite.py runs
the reference's own test files against this package.
"""

import importlib
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
_CANDIDATES = [os.environ.get("OCTFIELD_REF_SRC", ""), os.path.join(_ROOT, "baseline", "_ref", "octfield"),
               "/root/reference/pkg/src/octfield"]
REFERENCE_SRC = next((p for p in _CANDIDATES if p and os.path.exists(os.path.join(p, "__init__.py"))), None)
if REFERENCE_SRC is None:
    raise ImportError("octfield shim: reference sources not found (set OCTFIELD_REF_SRC)")
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

SWAPPED = ("errors", "octree", "field", "traversal", "render", "trainer", "modelio", "metrics")
for _name in SWAPPED:
    _mod = importlib.import_module("paper_2101_10994_b200." + _name)
    sys.modules[__name__ + "." + _name] = _mod
    globals()[_name] = _mod

# the remaining submodules (geometry, sampling, cli) load from the reference
# directory as octfield.<name>
__path__ = [REFERENCE_SRC]

with open(os.path.join(REFERENCE_SRC, "__init__.py")) as _fh:
    exec(compile(_fh.read(), os.path.join(REFERENCE_SRC, "__init__.py"), "exec"), globals())
