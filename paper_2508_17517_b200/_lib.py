"""ctypes binding of libairg.so (the C ABI declared in include/airg.h).

There is no fallback: importing the package on a machine without the built
library, or calling a kernel without a CUDA device, raises immediately.
"""

import ctypes as C
import os
import re

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, 'libairg.so')
HEADER = os.path.join(os.path.dirname(HERE), 'include', 'airg.h')

OK, ERR_ARG, ERR_CUDA, ERR_VALUE, ERR_DIVERGED = 0, 1, 2, 3, 4

_lib = None

vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
f64 = C.c_double


class AirgError(RuntimeError):
    pass


def load():
    """Load libairg.so (building it first if it is missing and nvcc is present)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from .build_lib import build
        build()
    _lib = C.CDLL(LIB_PATH)
    _declare(_lib)
    return _lib


def header_symbols():
    """Function names declared in include/airg.h."""
    txt = open(HEADER).read()
    txt = re.sub(r'/\*.*?\*/', '', txt, flags=re.S)
    return sorted(set(re.findall(r'\b(airg_[a-z0-9_]+)\s*\(', txt)))


_SIGS = {}


def sig(name, *args, ret=C.c_int):
    _SIGS[name] = (ret, list(args))


def _declare(lib):
    for name, (ret, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = ret
        fn.argtypes = args


def last_error():
    lib = load()
    buf = C.create_string_buffer(4096)
    lib.airg_last_error(buf, 4096)
    return buf.value.decode(errors='replace')


def check(status, what=''):
    if status == OK:
        return
    msg = last_error()
    if status in (ERR_VALUE, ERR_ARG):
        raise ValueError(msg)
    raise AirgError(f'{what}: status {status}: {msg}')


def call(name, *args):
    lib = load()
    st = getattr(lib, name)(*args)
    check(st, name)
    return st


def ptr(t):
    """Device pointer of a torch tensor (or None -> NULL)."""
    if t is None:
        return None
    return vp(t.data_ptr())


def hptr(a):
    """Host pointer of a contiguous numpy array (or None -> NULL)."""
    if a is None:
        return None
    return vp(a.ctypes.data)


def stream_handle():
    import torch
    return vp(torch.cuda.current_stream().cuda_stream)


# ---- signatures (mirror include/airg.h) ---------------------------------
sig('airg_version')
sig('airg_last_error', C.c_char_p, C.c_int)
sig('airg_sm_count')
sig('airg_spmv', i32, vp, vp, vp, vp, vp, C.c_int, vp)
sig('airg_norm2', i32, vp, vp, vp)
sig('airg_poly_apply', C.c_int, i32, vp, vp, vp, C.c_int, vp, C.c_int, vp, vp, vp, vp, vp, vp,
    vp)
sig('airg_plan_create', C.c_int, C.POINTER(vp))
sig('airg_plan_destroy', vp)
sig('airg_plan_set_top', vp, i32, vp, vp, vp)
sig('airg_plan_set_level', vp, C.c_int, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
    C.c_int, C.c_int, vp, vp, i64, vp, vp, vp)
sig('airg_plan_set_coarse', vp, i32, vp, vp, vp, C.c_int, C.c_int, vp, C.c_int, vp, vp, vp, vp)
sig('airg_plan_vcycle', vp, C.c_int, vp, vp, C.c_int, vp)
sig('airg_plan_richardson', vp, vp, vp, f64, f64, C.c_int, C.c_int, vp, vp, vp, vp)
sig('airg_plan_launches', vp, ret=i64)


def as_f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def as_i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)
