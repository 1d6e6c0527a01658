# mpmm/_kernels_cuda.py -- reference-side binding of libmpmm_cuda.so
import ctypes, os
import numpy as np

NAME = "cuda"
_lib = ctypes.CDLL(os.environ.get("MPMM_CUDA_LIB", "libmpmm_cuda.so"))
_D, _I = ctypes.POINTER(ctypes.c_double), ctypes.c_int64
_lib.mpmm_last_error.restype = ctypes.c_char_p
for f in ("dd_simple_rows", "qd_simple_rows"):
    getattr(_lib, "mpmm_" + f).argtypes = [_D, _D, _D, _I, _I, _I, _I, _I]
for f in ("dd_block_cells", "qd_block_cells"):
    getattr(_lib, "mpmm_" + f).argtypes = [_D, _D, _D, _I, _I, _I, _I, _I, _I]
for f in ("dd_ewise_add", "dd_ewise_sub", "qd_ewise_add", "qd_ewise_sub"):
    getattr(_lib, "mpmm_" + f).argtypes = [_D, _D, _D, _I, _I, _I, _I]

def _p(x):
    # the reference's buffers are C-contiguous float64 (matrix.py:47-48)
    assert x.dtype == np.float64 and x.flags.c_contiguous
    return x.ctypes.data_as(_D)

def _ok(rc):
    if rc:
        raise (ValueError if rc == 1 else RuntimeError)(_lib.mpmm_last_error().decode())

def dd_simple_rows(a, b, c, i0, i1):        # _kernels.pyx:36
    _ok(_lib.mpmm_dd_simple_rows(_p(a), _p(b), _p(c), a.shape[0], a.shape[1], b.shape[1], i0, i1))
def qd_simple_rows(a, b, c, i0, i1):        # _kernels.pyx:344
    _ok(_lib.mpmm_qd_simple_rows(_p(a), _p(b), _p(c), a.shape[0], a.shape[1], b.shape[1], i0, i1))
def dd_block_cells(a, b, c, n_min, c0, c1): # _kernels.pyx:103
    _ok(_lib.mpmm_dd_block_cells(_p(a), _p(b), _p(c), a.shape[0], a.shape[1], b.shape[1], n_min, c0, c1))
def qd_block_cells(a, b, c, n_min, c0, c1): # _kernels.pyx:366
    _ok(_lib.mpmm_qd_block_cells(_p(a), _p(b), _p(c), a.shape[0], a.shape[1], b.shape[1], n_min, c0, c1))
def dd_ewise_add(x, y, o, i0, i1):          # _kernels.pyx:207
    _ok(_lib.mpmm_dd_ewise_add(_p(x), _p(y), _p(o), x.shape[0], x.shape[1], i0, i1))
def dd_ewise_sub(x, y, o, i0, i1):          # _kernels.pyx:220
    _ok(_lib.mpmm_dd_ewise_sub(_p(x), _p(y), _p(o), x.shape[0], x.shape[1], i0, i1))
def qd_ewise_add(x, y, o, i0, i1):          # _kernels.pyx:407
    _ok(_lib.mpmm_qd_ewise_add(_p(x), _p(y), _p(o), x.shape[0], x.shape[1], i0, i1))
def qd_ewise_sub(x, y, o, i0, i1):          # _kernels.pyx:431
    _ok(_lib.mpmm_qd_ewise_sub(_p(x), _p(y), _p(o), x.shape[0], x.shape[1], i0, i1))
