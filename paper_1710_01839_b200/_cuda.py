"""ctypes binding of ``libmpmm_cuda.so`` (C ABI: ``include/mpmm_cuda.h``).

This module is the ``cuda`` kernel backend.  Its module-level ``NAME`` and
eight range functions follow the reference's kernel-module protocol
(``pkg/src/mpmm/backend.py:28-30``; signatures of ``_kernels.pyx:36-452``):
numpy ``(rows, cols, comps)`` float64 C-contiguous arrays in, results
written in place, nothing returned.  The ``*_dev`` wrappers take raw device
pointers (``torch.Tensor.data_ptr()``) for the device-resident paths.

There is no CPU fallback: if the library cannot be loaded, every entry
point raises :class:`~paper_1710_01839_b200.errors.DeviceError`.
"""

import ctypes
import os
import threading

import numpy as np

from .errors import DeviceError, ShapeError

NAME = "cuda"

_HERE = os.path.dirname(os.path.abspath(__file__))
# MPMM_LIB_PATH: load a variant build instead (tools/ experiments only)
LIB_PATH = os.environ.get("MPMM_LIB_PATH") or os.path.join(_HERE, "libmpmm_cuda.so")

_lib = None
_load_error = None

_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_int64
_INT = ctypes.c_int
_VP = ctypes.c_void_p

# (name, argtypes) for every symbol declared in include/mpmm_cuda.h
_SIGNATURES = {
    "mpmm_abi_version": [],
    "mpmm_last_error": [],
    "mpmm_set_device": [_INT],
    "mpmm_device_count": [ctypes.POINTER(_INT)],
    "mpmm_tile_for_nmin": [_I64, ctypes.POINTER(_INT), ctypes.POINTER(_INT)],
    "mpmm_gemm_geometry": [_INT, _INT, _I64] + [ctypes.POINTER(_INT)] * 5,
    "mpmm_dd_simple_rows": [_D, _D, _D, _I64, _I64, _I64, _I64, _I64],
    "mpmm_qd_simple_rows": [_D, _D, _D, _I64, _I64, _I64, _I64, _I64],
    "mpmm_dd_block_cells": [_D, _D, _D, _I64, _I64, _I64, _I64, _I64, _I64],
    "mpmm_qd_block_cells": [_D, _D, _D, _I64, _I64, _I64, _I64, _I64, _I64],
    "mpmm_dd_ewise_add": [_D, _D, _D, _I64, _I64, _I64, _I64],
    "mpmm_dd_ewise_sub": [_D, _D, _D, _I64, _I64, _I64, _I64],
    "mpmm_qd_ewise_add": [_D, _D, _D, _I64, _I64, _I64, _I64],
    "mpmm_qd_ewise_sub": [_D, _D, _D, _I64, _I64, _I64, _I64],
    "mpmm_gemm_host": [_INT, _INT, _I64, _I64, _I64, _I64, _D, _D, _D, _INT,
                       ctypes.POINTER(_INT)],
    "mpmm_gemm_dev": [_INT, _INT, _I64, _I64, _I64, _I64, _VP, _I64, _VP, _I64, _VP, _I64,
                      _INT, _VP, _VP],
    "mpmm_gemm_batched_dev": [_INT, _INT, _I64, _I64, _I64, _I64, _I64, _VP, _INT, _VP, _VP],
    "mpmm_ewise_batched_dev": [_INT, _I64, _I64, _I64, _VP, _VP],
    "mpmm_block_cells_dev": [_INT, _I64, _I64, _I64, _I64, _I64, _I64, _VP, _I64, _VP, _I64,
                             _VP, _I64, _VP],
    "mpmm_ewise_dev": [_INT, _INT, _I64, _I64, _VP, _I64, _VP, _I64, _INT, _VP, _I64, _INT,
                       _VP, _I64, _INT, _VP, _I64, _VP],
    "mpmm_nonfinite_dev": [_INT, _I64, _I64, _VP, _I64, _VP, _VP],
    "mpmm_fp64_burn_dev": [_INT, _INT, _INT, _I64, _VP, _VP],
    "mpmm_gen_inputs_dev": [_INT, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                            ctypes.c_uint64, ctypes.c_uint64, _I64, _I64, _VP, _VP],
    "mpmm_oz_scan_dev": [_INT, _INT, _I64, _I64, _VP, _I64, _VP, _VP, _VP],
    "mpmm_oz_residues_dev": [_INT, _INT, _INT, _INT, _I64, _I64, _VP, _I64, _VP, _INT, _INT,
                             _VP, _I64, _I64, _VP],
    "mpmm_oz_plan": [_INT, _I64, _I64, _I64, _VP, _VP, ctypes.POINTER(_INT), _VP,
                     ctypes.POINTER(_INT), _VP, _VP, ctypes.POINTER(_INT), _VP, _VP],
    "mpmm_gemm_exact_dev": [_INT, _I64, _I64, _I64, _VP, _I64, _VP, _I64, _VP, _I64, _VP],
    "mpmm_exact_release": [],
    "mpmm_residue_gemm_dev": [_I64, _I64, _I64, _I64, _VP, _VP, _VP, _VP],
    "mpmm_int8_gemm_batched_dev": [_I64, _I64, _I64, _I64, _VP, _VP, _VP, _VP, _I64, _VP],
    "mpmm_oz_combine_dev": [_INT, _VP, _INT, _I64, _I64, _VP, _VP, _VP],
    "mpmm_oz_shifts_dev": [_INT, _INT, _VP, _I64, _VP, _VP, _VP, _VP],
    "mpmm_exact_check_dev": [_INT, _I64, _I64, _I64, _VP, _I64, _VP, _I64, _VP, _I64, _VP, _VP,
                             _I64, _INT, _VP, _VP],
    "mpmm_ipc_handle_size": [],
    "mpmm_ipc_alloc": [_I64, _VP, ctypes.POINTER(_VP), _VP],
    "mpmm_ipc_free": [_VP],
    "mpmm_ipc_open": [_VP, ctypes.POINTER(_VP)],
    "mpmm_ipc_close": [_VP],
    "mpmm_peer_last_error": [],
    "mpmm_multi_plan": [_I64, _I64, _INT, _I64, _VP, _VP, ctypes.POINTER(_INT)],
    "mpmm_strassen_dev": [_INT, _I64, _I64, _I64, _I64, _I64, _VP, _I64, _VP, _I64, _VP, _I64,
                          _VP, _VP, _VP],
    "mpmm_init": [_INT, _VP],
    "mpmm_finalize": [],
    "mpmm_runtime_gpus": [ctypes.POINTER(_INT), _VP, _INT],
    "mpmm_gemm_multi": [_INT, _INT, _I64, _I64, _I64, _I64, _I64, _D, _D, _D, _I64,
                        ctypes.POINTER(_INT), ctypes.POINTER(ctypes.c_double)],
    "mpmm_timer_create": [ctypes.POINTER(_VP)],
    "mpmm_timer_start": [_VP, _VP],
    "mpmm_timer_stop": [_VP, _VP],
    "mpmm_timer_elapsed_ms": [_VP, ctypes.POINTER(ctypes.c_float)],
    "mpmm_timer_destroy": [_VP],
    "mpmm_host_frobenius_norm": [_INT, _D, _I64, _D],
    "mpmm_host_frobenius_rel_diff": [_INT, _D, _D, _I64, _D],
}

ALGO_SIMPLE = 0
ALGO_BLOCK = 1
ALGO_BLOCK_FAST = 2   # opt-in faithful DD sequence (not bit-identical)
ALGO_STRASSEN = 3     # mpmm_gemm_multi only


def load():
    """Load the library once; raise DeviceError when it is missing."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is not None:
        raise DeviceError(_load_error)
    if not os.path.exists(LIB_PATH):
        # not cached: build() may produce the library later in this process
        raise DeviceError(f"CUDA extension not built: {LIB_PATH} is missing "
                          "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as ex:
        _load_error = f"cannot load {LIB_PATH}: {ex}"
        raise DeviceError(_load_error) from None
    for name, argtypes in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = (ctypes.c_char_p if name in ("mpmm_last_error", "mpmm_peer_last_error")
                      else ctypes.c_int)
    _lib = lib
    return lib


def available():
    try:
        load()
        return True
    except DeviceError:
        return False


def exported_symbols():
    return list(_SIGNATURES)


_tls = threading.local()


def sync_device():
    """Mirror torch's current device into the library's runtime (once per
    change, per host thread)."""
    import torch
    dev = torch.cuda.current_device()
    if getattr(_tls, "device", None) != dev:
        check(load().mpmm_set_device(dev))
        _tls.device = dev


def check(rc):
    if rc != 0:
        msg = load().mpmm_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(msg)
        raise DeviceError(msg)


def device_count():
    n = ctypes.c_int(0)
    check(load().mpmm_device_count(ctypes.byref(n)))
    return n.value


def tile_for_nmin(n_min):
    t, s = ctypes.c_int(0), ctypes.c_int(0)
    check(load().mpmm_tile_for_nmin(n_min, ctypes.byref(t), ctypes.byref(s)))
    return t.value, s.value


def gemm_geometry(comps, algo, n_min):
    """dict(tile_m, tile_n, threads, ctas_per_sm, sm_count) on the current device."""
    vals = [ctypes.c_int(0) for _ in range(5)]
    check(load().mpmm_gemm_geometry(comps, algo, n_min, *[ctypes.byref(v) for v in vals]))
    keys = ("tile_m", "tile_n", "threads", "ctas_per_sm", "sm_count")
    return dict(zip(keys, (v.value for v in vals)))


# ---------------------------------------------------------------------------
# reference kernel-module protocol (host numpy arrays)
# ---------------------------------------------------------------------------

def _arr(x, comps):
    if not isinstance(x, np.ndarray) or x.dtype != np.float64 or x.ndim != 3 \
            or not x.flags.c_contiguous:
        raise TypeError("expected a C-contiguous float64 (rows, cols, comps) array")
    if x.shape[2] != comps:
        raise ShapeError(f"expected {comps} components, got {x.shape[2]}")
    return x.ctypes.data_as(_D)


def _simple(comps, fn, a, b, c, i0, i1):
    sync_device()
    m, l = a.shape[0], a.shape[1]
    n = b.shape[1]
    check(fn(_arr(a, comps), _arr(b, comps), _arr(c, comps), m, l, n, i0, i1))


def _cells(comps, fn, a, b, c, n_min, cell0, cell1):
    sync_device()
    m, l = a.shape[0], a.shape[1]
    n = b.shape[1]
    check(fn(_arr(a, comps), _arr(b, comps), _arr(c, comps), m, l, n, n_min, cell0, cell1))


def _ew(comps, fn, x, y, out, i0, i1):
    sync_device()
    check(fn(_arr(x, comps), _arr(y, comps), _arr(out, comps), x.shape[0], x.shape[1], i0, i1))


def dd_simple_rows(a, b, c, i0, i1):
    """_kernels.pyx:36-100 on the GPU."""
    _simple(2, load().mpmm_dd_simple_rows, a, b, c, i0, i1)


def qd_simple_rows(a, b, c, i0, i1):
    """_kernels.pyx:344-363 on the GPU."""
    _simple(4, load().mpmm_qd_simple_rows, a, b, c, i0, i1)


def dd_block_cells(a, b, c, n_min, cell0, cell1):
    """_kernels.pyx:103-186 on the GPU (accumulates into c)."""
    _cells(2, load().mpmm_dd_block_cells, a, b, c, n_min, cell0, cell1)


def qd_block_cells(a, b, c, n_min, cell0, cell1):
    """_kernels.pyx:366-404 on the GPU (accumulates into c)."""
    _cells(4, load().mpmm_qd_block_cells, a, b, c, n_min, cell0, cell1)


def dd_ewise_add(x, y, out, i0, i1):
    _ew(2, load().mpmm_dd_ewise_add, x, y, out, i0, i1)


def dd_ewise_sub(x, y, out, i0, i1):
    _ew(2, load().mpmm_dd_ewise_sub, x, y, out, i0, i1)


def qd_ewise_add(x, y, out, i0, i1):
    _ew(4, load().mpmm_qd_ewise_add, x, y, out, i0, i1)


def qd_ewise_sub(x, y, out, i0, i1):
    _ew(4, load().mpmm_qd_ewise_sub, x, y, out, i0, i1)


# ---------------------------------------------------------------------------
# device-resident entry points (raw pointers, element leading dimensions)
# ---------------------------------------------------------------------------

def gemm_host(comps, algo, n_min, a, b, c, accumulate=False):
    """c = a*b (or c += a*b) for host arrays through the pipelined C-ABI
    entry; returns True when every output component is finite."""
    sync_device()
    flag = ctypes.c_int(0)
    check(load().mpmm_gemm_host(comps, algo, n_min, a.shape[0], a.shape[1], b.shape[1],
                                _arr(a, comps), _arr(b, comps), _arr(c, comps),
                                1 if accumulate else 0, ctypes.byref(flag)))
    return flag.value == 0


def gemm_dev(comps, algo, n_min, m, l, n, A, lda, B, ldb, C, ldc, accumulate,
             nonfinite=None, stream=None):
    sync_device()
    check(load().mpmm_gemm_dev(comps, algo, n_min, m, l, n, A, lda, B, ldb, C, ldc,
                               1 if accumulate else 0, nonfinite, stream))


def gemm_batched_dev(comps, algo, n_min, batch, m, l, n, problems, accumulate, nonfinite=None,
                     stream=None):
    """``problems``: device pointer to ``batch`` x 6 int64 {A, B, C, lda, ldb, ldc}."""
    sync_device()
    check(load().mpmm_gemm_batched_dev(comps, algo, n_min, batch, m, l, n, problems,
                                       1 if accumulate else 0, nonfinite, stream))


def ewise_batched_dev(comps, batch, rows, cols, problems, stream=None):
    """``problems``: device pointer to ``batch`` x 14 int64 (see mpmm_cuda.h)."""
    sync_device()
    check(load().mpmm_ewise_batched_dev(comps, batch, rows, cols, problems, stream))


def strassen_dev(comps, cutoff, leaf_n_min, m, l, n, A, lda, B, ldb, C, ldc, nonfinite=None,
                 stats=None, stream=None):
    """``stats``: optional ctypes int64[2] receiving {multiplications, additions}."""
    sync_device()
    check(load().mpmm_strassen_dev(comps, cutoff, leaf_n_min, m, l, n, A, lda, B, ldb, C, ldc,
                                   nonfinite, stats, stream))


def runtime_init(ngpus, devices=None):
    """Single-process multi-GPU runtime (NCCL communicators owned by the library).
    torch is imported first so the library binds the NCCL build torch uses."""
    import torch  # noqa: F401
    arr = None
    if devices is not None:
        arr = (ctypes.c_int * len(devices))(*devices)
        ngpus = len(devices)
    check(load().mpmm_init(ngpus, ctypes.cast(arr, ctypes.c_void_p) if arr else None))


def runtime_finalize():
    check(load().mpmm_finalize())


def runtime_gpus():
    n = _INT(0)
    ids = (ctypes.c_int * 64)()
    check(load().mpmm_runtime_gpus(ctypes.byref(n), ctypes.cast(ids, ctypes.c_void_p), 64))
    return list(ids[:n.value])


def exact_release():
    """mpmm_exact_release: drop the exact mode's cached plans and buffers."""
    check(load().mpmm_exact_release())


def _peer_check(rc):
    if rc:
        raise DeviceError(load().mpmm_peer_last_error().decode() or f"peer error {rc}")


def ipc_alloc(nbytes, init=None):
    """(device pointer, IPC handle bytes) of a fresh cudaMalloc'ed buffer,
    filled from the pointer ``init`` when given."""
    size = load().mpmm_ipc_handle_size()
    handle = ctypes.create_string_buffer(size)
    ptr = ctypes.c_void_p()
    _peer_check(load().mpmm_ipc_alloc(nbytes, init, ctypes.byref(ptr), handle))
    return ptr.value, handle.raw


def ipc_open(handle):
    buf = ctypes.create_string_buffer(handle, len(handle))
    ptr = ctypes.c_void_p()
    _peer_check(load().mpmm_ipc_open(buf, ctypes.byref(ptr)))
    return ptr.value


def ipc_close(ptr):
    _peer_check(load().mpmm_ipc_close(ptr))


def ipc_free(ptr):
    _peer_check(load().mpmm_ipc_free(ptr))


def multi_plan(m, l, ngpus, panels=0):
    """mpmm_gemm_multi's schedule: ([(r0, r1)] per GPU, [(k0, k1)] per
    k-panel).  Pure host code: works without a GPU."""
    rows = (ctypes.c_int64 * (2 * ngpus))()
    kb = (ctypes.c_int64 * (max(l, 1) + 2))()
    npan = _INT(0)
    if load().mpmm_multi_plan(m, l, ngpus, panels, ctypes.cast(rows, _VP), ctypes.cast(kb, _VP),
                              ctypes.byref(npan)):
        raise ValueError("bad multi-GPU plan request")
    return ([(rows[2 * g], rows[2 * g + 1]) for g in range(ngpus)],
            [(kb[p], kb[p + 1]) for p in range(npan.value)])


def gemm_multi(comps, algo, n_min, cutoff, a, b, c, panels=0):
    """c = a*b (host float64 arrays (m,l,comps) / (l,n,comps) / (m,n,comps)) on
    the runtime's GPUs; returns (nonfinite, device_ms)."""
    m, l, n = a.shape[0], a.shape[1], b.shape[1]
    bad, ms = _INT(0), ctypes.c_double(0.0)
    check(load().mpmm_gemm_multi(comps, algo, n_min, cutoff, m, l, n, _arr(a, comps),
                                 _arr(b, comps), _arr(c, comps), panels, ctypes.byref(bad),
                                 ctypes.byref(ms)))
    return bool(bad.value), ms.value


class Timer:
    """Device event timer (mpmm_timer_*), start/stop on a stream."""

    def __init__(self):
        self._t = ctypes.c_void_p()
        check(load().mpmm_timer_create(ctypes.byref(self._t)))

    def start(self, stream=None):
        check(load().mpmm_timer_start(self._t, stream))

    def stop(self, stream=None):
        check(load().mpmm_timer_stop(self._t, stream))

    def elapsed_ms(self):
        ms = ctypes.c_float(0.0)
        check(load().mpmm_timer_elapsed_ms(self._t, ctypes.byref(ms)))
        return ms.value

    def __del__(self):
        if getattr(self, "_t", None) and _lib is not None:
            _lib.mpmm_timer_destroy(self._t)
            self._t = None


def block_cells_dev(comps, n_min, cell0, cell1, m, l, n, A, lda, B, ldb, C, ldc, stream=None):
    sync_device()
    check(load().mpmm_block_cells_dev(comps, n_min, cell0, cell1, m, l, n, A, lda, B, ldb,
                                      C, ldc, stream))


def ewise_dev(comps, rows, cols, O, ldo, X, ldx, Y, ldy, sy, Z=None, ldz=0, sz=1, W=None,
              ldw=0, sw=1, stream=None):
    nops = 1 + (Z is not None) + (W is not None)
    sync_device()
    check(load().mpmm_ewise_dev(comps, nops, rows, cols, X, ldx, Y, ldy, sy, Z, ldz, sz,
                                W, ldw, sw, O, ldo, stream))


def nonfinite_dev(comps, rows, cols, X, ldx, flag, stream=None):
    sync_device()
    check(load().mpmm_nonfinite_dev(comps, rows, cols, X, ldx, flag, stream))


def exact_check_dev(comps, m, l, n, A, lda, B, ldb, C, ldc, idx_i, idx_j, count, u_exp, ratio,
                    stream=None):
    sync_device()
    check(load().mpmm_exact_check_dev(comps, m, l, n, A, lda, B, ldb, C, ldc, idx_i, idx_j,
                                      count, u_exp, ratio, stream))


def gen_inputs_dev(comps, state, inc, first_draw, rows, cols, out, stream=None):
    sync_device()
    m64 = (1 << 64) - 1
    check(load().mpmm_gen_inputs_dev(comps, state >> 64, state & m64, inc >> 64, inc & m64,
                                     first_draw, rows, cols, out, stream))


def oz_scan_dev(by_cols, comps, rows, cols, X, ld, EL, status, stream=None):
    sync_device()
    check(load().mpmm_oz_scan_dev(by_cols, comps, rows, cols, X, ld, EL, status, stream))


def oz_residues_dev(by_cols, comps, c0, c1, rows, cols, X, ld, shift, nmod, words, R, rpitch,
                    rplane, stream=None):
    sync_device()
    check(load().mpmm_oz_residues_dev(by_cols, comps, c0, c1, rows, cols, X, ld, shift, nmod,
                                      words, R, rpitch, rplane, stream))


def gemm_exact_dev(comps, m, l, n, A, lda, B, ldb, C, ldc, stream=None):
    """Returns 0, or MPMM_ERR_RANGE (4) / MPMM_ERR_NONFINITE (5) with the
    message in last_error(); raises on other failures."""
    sync_device()
    rc = load().mpmm_gemm_exact_dev(comps, m, l, n, A, lda, B, ldb, C, ldc, stream)
    if rc in (4, 5):
        return rc
    check(rc)
    return 0


def residue_gemm_dev(m, n, k, batch, A, Bt, R, stream=None):
    sync_device()
    check(load().mpmm_residue_gemm_dev(m, n, k, batch, A, Bt, R, stream))


def last_error():
    return load().mpmm_last_error().decode(errors="replace")


def oz_plan(comps, m, n, l, ela, elb):
    """Host planner (no device work): returns (jobs int32[njobs, 8],
    ranges_a, shift_a[na, m], ranges_b, shift_b[nb, n]) or None when no
    split is representable."""
    ela = np.ascontiguousarray(ela, dtype=np.int32)
    elb = np.ascontiguousarray(elb, dtype=np.int32)
    jobs = np.zeros((16, 8), dtype=np.int32)
    ra, rb = np.zeros(8, dtype=np.int32), np.zeros(8, dtype=np.int32)
    sa, sb = np.zeros((4, max(m, 1)), dtype=np.int32), np.zeros((4, max(n, 1)), dtype=np.int32)
    nj, na, nb = _INT(0), _INT(0), _INT(0)
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    rc = load().mpmm_oz_plan(comps, m, n, l, vp(ela), vp(elb), ctypes.byref(nj), vp(jobs),
                             ctypes.byref(na), vp(ra), vp(sa), ctypes.byref(nb), vp(rb), vp(sb))
    if rc == 4:
        return None
    check(rc)
    return (jobs[:nj.value], ra[:2 * na.value].reshape(-1, 2), sa[:na.value, :m],
            rb[:2 * nb.value].reshape(-1, 2), sb[:nb.value, :n])


def int8_gemm_batched_dev(m, n, k, batch, A, Bt, C, workspace, ws_bytes, stream=None):
    sync_device()
    check(load().mpmm_int8_gemm_batched_dev(m, n, k, batch, A, Bt, C, workspace, ws_bytes,
                                            stream))


def oz_combine_dev(comps, jobs, njobs, m, n, C, status, stream=None):
    """jobs: host pointer to njobs 56-byte CrtJob records."""
    sync_device()
    check(load().mpmm_oz_combine_dev(comps, jobs, njobs, m, n, C, status, stream))


def oz_shifts_dev(comps, ranges, odim, EL, shift, beta, stream=None):
    """ranges: sequence of (c0, c1) component ranges (<= 4)."""
    sync_device()
    flat = (ctypes.c_int * (2 * len(ranges)))(*[c for r in ranges for c in r])
    check(load().mpmm_oz_shifts_dev(comps, len(ranges), ctypes.cast(flat, ctypes.c_void_p),
                                    odim, EL, shift, beta, stream))


def fp64_burn_dev(op, blocks, threads, iters, scratch, stream=None):
    sync_device()
    check(load().mpmm_fp64_burn_dev(op, blocks, threads, iters, scratch, stream))


def host_frobenius_norm(comps, x):
    out = ctypes.c_double(0.0)
    x = np.ascontiguousarray(x, dtype=np.float64)
    return load().mpmm_host_frobenius_norm(comps, x.ctypes.data_as(_D), x.size // comps,
                                           ctypes.byref(out)), out.value


def host_frobenius_rel_diff(comps, x, y):
    out = ctypes.c_double(0.0)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return load().mpmm_host_frobenius_rel_diff(comps, x.ctypes.data_as(_D), y.ctypes.data_as(_D),
                                               x.size // comps, ctypes.byref(out)), out.value
