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


CALL_TIMES = {} if os.environ.get('AIRG_PROFILE_CALLS') else None


def call(name, *args):
    lib = load()
    if CALL_TIMES is None:
        st = getattr(lib, name)(*args)
    else:
        import time
        t0 = time.perf_counter()
        st = getattr(lib, name)(*args)
        rec = CALL_TIMES.setdefault(name, [0, 0.0])
        rec[0] += 1
        rec[1] += time.perf_counter() - t0
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
    """Raw cudaStream_t of torch's current stream on the current device.
    (torch.cuda.current_stream() costs ~16 us per call in device-index
    bookkeeping; the setup makes thousands of library calls.)"""
    import torch
    C_ = torch._C
    return vp(C_._cuda_getCurrentRawStream(C_._cuda_getDevice()))


# ---- signatures (mirror include/airg.h) ---------------------------------
sig('airg_version')
sig('airg_last_error', C.c_char_p, C.c_int)
sig('airg_sm_count')
sig('airg_spmv', i32, vp, vp, vp, vp, vp, C.c_int, vp)
sig('airg_csr_to_ell', i32, vp, vp, vp, C.c_int, vp, vp, vp)
sig('airg_spmv_ell', i32, C.c_int, vp, vp, vp, vp, C.c_int, vp)
sig('airg_norm2', i32, vp, vp, vp)
sig('airg_poly_apply', C.c_int, i32, vp, vp, vp, C.c_int, vp, C.c_int, vp, vp, vp, vp, vp, vp,
    C.c_int, vp)
sig('airg_plan_set_exact', vp, C.c_int)
sig('airg_plan_create', C.c_int, C.POINTER(vp))
sig('airg_plan_destroy', vp)
sig('airg_plan_set_top', vp, i32, vp, vp, vp)
sig('airg_plan_set_level', vp, C.c_int, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
    C.c_int, C.c_int, vp, vp, i64, vp, vp, vp)
sig('airg_plan_set_coarse', vp, i32, vp, vp, vp, C.c_int, C.c_int, vp, C.c_int, vp, vp, vp, vp)
sig('airg_plan_vcycle', vp, C.c_int, vp, vp, C.c_int, vp)
sig('airg_plan_richardson', vp, vp, vp, f64, f64, C.c_int, C.c_int, vp, vp, vp, vp)
sig('airg_plan_launches', vp, ret=i64)
sig('airg_plan_coarse_mode', vp)
sig('airg_plan_graph_count', vp)
sig('airg_plan_staging', vp, C.POINTER(vp), C.POINTER(vp))
sig('airg_copy_d2d', vp, vp, i64, vp)
sig('airg_nccl_unique_id', C.c_char_p)
sig('airg_comm_create', C.c_char_p, C.c_int, C.c_int, C.POINTER(vp))
sig('airg_comm_destroy', vp)
sig('airg_dplan_create', vp, C.c_int, C.POINTER(vp))
sig('airg_dplan_set_halo', vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp)
sig('airg_dplan_set_level', vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, i64, vp, vp, vp,
    i64, vp, vp, vp, i64, vp, vp, C.c_int, vp)
sig('airg_dplan_set_top', vp, C.c_int, vp, vp, vp, i64)
sig('airg_dplan_set_dcoarse', vp, C.c_int, vp, vp, vp, i64, C.c_int, vp, vp, vp, C.c_int, vp, vp, vp)
sig('airg_dplan_finish', vp, vp, vp)
sig('airg_dplan_richardson', vp, vp, vp, f64, f64, C.c_int, vp, vp, vp, vp)
sig('airg_dplan_destroy', vp)
u64 = C.c_uint64
pp = C.POINTER(vp)
sig('airg_result_info', vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i64))
sig('airg_result_take', vp, vp, vp, vp, vp)
sig('airg_result_free', vp)
sig('airg_result_detach', vp, vp, vp, vp, vp)
sig('airg_buffer_free', vp, vp)
sig('airg_pcg64_fill', u64, u64, u64, u64, i64, f64, f64, vp, vp)
sig('airg_random_unit', u64, u64, u64, u64, i64, vp, vp, vp)
sig('airg_diagonal', i32, vp, vp, vp, vp, vp)
sig('airg_reserve', i64, vp)
sig('airg_advection_2d', i32, i32, f64, f64, vp, vp, vp, vp)
sig('airg_strength', i32, vp, vp, vp, i64, f64, pp, pp, vp)
sig('airg_pmisr', i32, vp, vp, u64, u64, u64, u64, C.c_int, vp, C.POINTER(i32), vp)
sig('airg_cf_pmisr', i32, vp, vp, vp, i64, f64, u64, u64, u64, u64, C.c_int, vp, C.POINTER(i32),
    vp)
sig('airg_ddc_pass', i32, vp, vp, vp, vp, f64, C.c_int, vp, vp)
sig('airg_split_index', i32, vp, vp, vp, vp, C.POINTER(i32), vp)
sig('airg_repair_split', i32, vp, vp, vp, C.POINTER(i32), vp)
sig('airg_prolong_onepoint', i32, vp, vp, vp, vp, vp, vp, vp)
sig('airg_spgemm', i32, i32, i32, vp, vp, vp, vp, vp, vp, C.c_int, pp, vp)
sig('airg_spgemm_masked', i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, pp, vp)
sig('airg_poly_assemble', i32, vp, vp, vp, C.c_int, vp, vp, vp, pp, vp)
sig('airg_neumann_base', i32, vp, vp, vp, vp, pp, vp)
sig('airg_scale_columns', i64, vp, vp, vp, vp)
sig('airg_drop_lump', i32, i32, vp, vp, vp, f64, C.c_int, pp, C.POINTER(i32), vp)
sig('airg_galerkin', i32, i32, vp, vp, vp, vp, vp, vp, vp, f64, C.c_int, pp, vp)
sig('airg_ap_onepoint', i32, i32, i32, vp, vp, vp, vp, pp, vp)
sig('airg_advection_dg', i32, i32, vp, C.c_int, C.c_int, pp, vp)
sig('airg_extract', i32, vp, vp, vp, vp, vp, i32, pp, vp)
sig('airg_extract_ex', i32, vp, vp, vp, vp, vp, i32, C.c_double, pp, vp)
sig('airg_label_colmap', i32, vp, C.c_int, vp, vp, vp)
sig('airg_restriction', i32, i32, vp, vp, vp, vp, vp, pp, vp)
sig('airg_arnoldi', i32, vp, vp, vp, vp, C.c_int, vp, C.POINTER(i32), C.POINTER(f64), vp)
sig('airg_advection_2d_rows', i32, i32, f64, f64, i64, i64, vp, vp, vp, C.POINTER(i64), vp)
sig('airg_strength_rows', i32, i32, vp, vp, vp, i64, f64, pp, vp)
sig('airg_union_rows', i32, vp, vp, vp, vp, pp, vp)
sig('airg_luby_weights', i32, i64, vp, u64, u64, u64, u64, vp, vp)
sig('airg_luby_round', i32, vp, vp, vp, vp, vp, C.c_int, C.c_int, C.POINTER(i32), vp)
sig('airg_luby_finish', i32, vp, vp, vp)
sig('airg_ddc_ratios', i32, i32, vp, vp, vp, vp, vp, vp, C.POINTER(i32), vp, vp)
sig('airg_ddc_hist', i32, vp, vp, C.c_int, vp, vp)
sig('airg_ddc_convert', i32, vp, vp, f64, C.c_int, vp, C.POINTER(i32), vp)
sig('airg_gather_int', i64, vp, vp, vp, vp)
sig('airg_pcg64_fill_at', u64, u64, u64, u64, i64, i64, f64, f64, vp, vp)
sig('airg_spgemm_ex', i32, i32, i32, vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, f64, C.c_int,
    C.c_int, pp, vp)
sig('airg_poly_assemble_ex', i32, i32, vp, vp, vp, vp, C.c_int, vp, vp, vp, pp, vp)


def pcg_params(seed):
    """(state_hi, state_lo, inc_hi, inc_lo) of numpy's PCG64(SeedSequence(seed))."""
    st = np.random.PCG64(np.random.SeedSequence(seed)).state['state']
    s, inc = int(st['state']), int(st['inc'])
    m = (1 << 64) - 1
    return s >> 64, s & m, inc >> 64, inc & m


def as_f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def as_i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)
