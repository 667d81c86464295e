"""ctypes binding of libhpgmxp.so (include/hpgmxp.h).

The library is built in-tree by ``python -m paper_2507_11512_b200.build`` (or
``__graft_entry__.build()``).  There is no fallback: if the shared object is
missing or fails to load, importing any device path raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# HPG_LIB: load another build of the same sources (A/B experiments)
LIB_PATH = os.environ.get("HPG_LIB") or os.path.join(HERE, "libhpgmxp.so")

F64 = 0
F32 = 1

E_ARG, E_CUDA, E_NCCL, E_COARSEN, E_UNSUPPORTED, E_SINGULAR = -1, -2, -3, -4, -5, -6

# every symbol include/hpgmxp.h declares: name -> (restype, argtypes)
_p = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_ip = C.POINTER(C.c_int)
_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)

SIGNATURES = {
    "hpg_abi_version": (_i, []),
    "hpg_last_error": (C.c_char_p, []),
    "hpg_host_level": (_i, [_ip, _ip, _ip, _dp, _i32p, _i32p, _i32p, _i64p, _i]),
    "hpg_host_send_rows": (_i64, [_ip, _ip, _ip, _i, _i, _i, _i64p]),
    "hpg_host_stage_offset": (_i64, [_ip, _ip, _i, _i, _i, _i, _i64p]),
    "hpg_nccl_unique_id": (_i, [_p, _i]),
    "hpg_create": (_i, [C.POINTER(_p), _i, _i, _i, _ip, _ip, _i, _i, _i, _i, _p, _p]),
    "hpg_destroy": (_i, [_p]),
    "hpg_stream": (_p, [_p]),
    "hpg_level_info": (_i, [_p, _i, _i64p, _i]),
    "hpg_export_level": (_i, [_p, _i, _dp, _i32p, _i32p, _i32p]),
    "hpg_export_f2c": (_i, [_p, _i, _i64p]),
    "hpg_set_coloring": (_i, [_p, _i, _i, _i64p, _i64p]),
    "hpg_jpl_color": (_i, [_i, _i, _i, _i, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), _i32p, _ip]),
    "hpg_spmv": (_i, [_p, _i, _i, _p, _p]),
    "hpg_exchange": (_i, [_p, _i, _i, _p]),
    "hpg_gs_sweep": (_i, [_p, _i, _i, _p, _p, _i]),
    "hpg_restrict": (_i, [_p, _i, _i, _p, _p, _p]),
    "hpg_prolong": (_i, [_p, _i, _i, _p, _p]),
    "hpg_vcycle": (_i, [_p, _i, _p, _p]),
    "hpg_cgs2": (_i, [_p, _i, _p, _i64, _i, _p, _p, _dp]),
    "hpg_cgs2_begin": (_i, [_p, _i, _p, _i64, _i, _p, _p]),
    "hpg_cgs2_end": (_i, [_p, _dp]),
    "hpg_gemv_combine": (_i, [_p, _i, _p, _i64, _i, _dp, _p]),
    "hpg_axpy_mixed": (_i, [_p, _i, _p, _p, _i64]),
    "hpg_residual": (_i, [_p, _p, _p, _p, _dp]),
    "hpg_scale_cast": (_i, [_p, _i, _p, C.c_double, _p, _i64]),
    "hpg_sumsq": (_i, [_p, _i, _p, _i64, _dp]),
    "hpg_sync": (_i, [_p]),
    "hpg_allreduce_host": (_i, [_p, _dp, _i]),
    "hpg_launch_count": (_i64, [_p]),
    "hpg_timers": (_i, [_p, _i, _dp]),
    "hpg_set_option": (_i, [_p, C.c_char_p, _i64]),
    "hpg_p2p_handle": (_i, [_p, _p, _i]),
    "hpg_p2p_open": (_i, [_p, _p, _i]),
}

_LIB = None


class HpgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libhpgmxp error {code}: {msg}")
        self.code = code


def lib():
    """Load (once) and return the CDLL; raises if the CUDA library is absent."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2507_11512_b200.build` "
                "(there is no CPU fallback)")
        # torch first: libhpgmxp's libnccl.so.2 dependency must bind to the NCCL
        # torch already loaded (same soname); loading the system NCCL first would
        # leave torch's libtorch_cuda with unresolved newer NCCL symbols.
        import torch  # noqa: F401
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def last_error():
    return lib().hpg_last_error().decode(errors="replace")


def check(code):
    """Map a C return code to the reference's exception classes."""
    if code == 0:
        return
    msg = last_error()
    if code == E_COARSEN:
        from .geometry import CoarseningError
        raise CoarseningError(msg)
    if code == E_NCCL:
        from .comm import ProtocolError
        raise ProtocolError(msg)
    if code == E_SINGULAR:
        from .smoother import SingularDiagonal
        raise SingularDiagonal(msg)
    if code in (E_ARG, E_UNSUPPORTED):
        raise ValueError(msg)
    raise HpgError(code, msg)


def ints(*v):
    return (C.c_int * len(v))(*v)


def ptr(t):
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def dptr(a):
    return a.ctypes.data_as(_dp)


def on_device(v, torch_dtype, device):
    """(device tensor, host array or None): a host numpy vector argument of the
    reference's array API is copied to the device; the caller copies results
    back into the host array (in-place contracts) -- compute stays on the GPU."""
    import numpy as np
    import torch
    if isinstance(v, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(v)).to(device=device, dtype=torch_dtype), v
    return v, None


def back_to_host(t, host):
    """Copy a device result into the caller's host array (if it gave one)."""
    if host is not None:
        host[...] = t.cpu().numpy().astype(host.dtype, copy=False)
