"""Kernel backend registry (reference ``pkg/src/mpmm/backend.py:1-56``).

The reference picks between its compiled Cython module (``ext``) and a
pure-Python mirror (``python``).  Here the product backend is ``cuda``:
the sm_100a kernels behind ``libmpmm_cuda.so`` (``_cuda.py``).  There is
deliberately no CPU fallback -- when the library is missing, ``kernels()``
raises :class:`DeviceError` instead of silently computing on the host.

``register()`` lets a caller add another module that follows the same
protocol (``NAME`` plus the eight range functions); the test-suite uses it
to plug the CPU oracle in for backend-equivalence checks, the way the
reference's tests switch between ``ext`` and ``python``
(tests/test_backend_equiv.py:31-69).
"""

import os
import warnings

from . import _cuda
from .errors import DeviceError

PROTOCOL = ("dd_simple_rows", "dd_block_cells", "dd_ewise_add", "dd_ewise_sub",
            "qd_simple_rows", "qd_block_cells", "qd_ewise_add", "qd_ewise_sub")

_registry = {"cuda": _cuda}
_active_name = "cuda"


def __getattr__(name):
    # HAVE_EXT is evaluated on first use, not at import: importing the
    # package must not map libmpmm_cuda.so (a CPU-only caller -- e.g. the
    # bench's reference arm -- imports helpers without touching the GPU)
    if name == "HAVE_EXT":
        return _cuda.available()
    raise AttributeError(name)


# The reference reads MPMM_BACKEND at import (backend.py:22-25): "python"
# forces its pure-Python kernels, anything else is ignored.  Neither CPU
# backend exists here, so the variable is ignored with a warning rather than
# making the package unimportable for environments that set it.
_env = os.environ.get("MPMM_BACKEND")
if _env and _env != "cuda":
    warnings.warn(f"MPMM_BACKEND={_env!r} ignored: this package ships only the 'cuda' "
                  "backend (no CPU kernels)", RuntimeWarning, stacklevel=2)


def kernels():
    """The active kernel module (raises DeviceError if it cannot load)."""
    mod = _registry[_active_name]
    if mod is _cuda:
        _cuda.load()
    return mod


def backend_name():
    return _registry[_active_name].NAME


def available_backends():
    names = [n for n, m in _registry.items() if m is not _cuda or _cuda.available()]
    return names


def register(name, module):
    """Add a protocol-conforming kernel module under ``name``."""
    missing = [f for f in PROTOCOL if not callable(getattr(module, f, None))]
    if missing or not hasattr(module, "NAME"):
        raise TypeError(f"backend {name!r} lacks {missing or ['NAME']}")
    _registry[name] = module


def unregister(name):
    global _active_name
    if name == "cuda":
        raise ValueError("the cuda backend cannot be removed")
    _registry.pop(name, None)
    if _active_name == name:
        _active_name = "cuda"


def use(name):
    """Switch the active backend; returns the previous name
    (reference backend.py:44-56).  Unknown names raise ValueError."""
    global _active_name
    if name not in _registry:
        raise ValueError(f"unknown backend {name!r}")
    if name == "cuda" and not _cuda.available():
        raise DeviceError("the CUDA kernels are not available in this install")
    prev = _registry[_active_name].NAME
    _active_name = name
    return prev


def is_cuda():
    return _registry[_active_name] is _cuda
