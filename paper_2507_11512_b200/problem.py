"""Device-resident 27-point ELL operands (ref: problem.py:31-175).

``EllMatrix`` here is a handle onto one level of a libhpgmxp hierarchy in one
precision: the values, int32 columns and the diagonal live in HBM in the
slot-major layout of csrc/hpg_kernels.cuh.  The reference's array fields
(``values``, ``col_idx``, ``row_nnz``, ``diag_pos``) are still available, as
host copies exported in the reference's row-major layout, so callers and the
parity tests can inspect exactly what the kernels use.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib

STENCIL_WIDTH = 27
PAD = -1
UNRESOLVED = -2


class EllMatrix:
    def __init__(self, ctx, level, prec):
        self.ctx = ctx
        self.level = level
        self.prec = prec
        info = ctx.level_info(level)
        self.n_rows = info["n"]
        self.width = STENCIL_WIDTH
        self.nnz_total = info["nnz"]
        self.n_cols_extended = info["n_ext"]
        self._host = None

    @property
    def implicit_nnz(self):
        """Nonzeros of the rows whose columns the kernels compute in closed form
        (implicit-index rows: 27 each, no column-index load) -- 0 with stencil off."""
        if not self.ctx.option("stencil"):
            return 0
        return 27 * self.ctx.level_info(self.level)["stencil_rows"]

    @property
    def dtype(self):
        return np.dtype(np.float32 if self.prec == _lib.F32 else np.float64)

    @property
    def torch_dtype(self):
        import torch
        return torch.float32 if self.prec == _lib.F32 else torch.float64

    def _export(self):
        if self._host is None:
            n = self.n_rows
            vals = np.zeros((n, STENCIL_WIDTH))
            cols = np.zeros((n, STENCIL_WIDTH), dtype=np.int32)
            nnz = np.zeros(n, dtype=np.int32)
            diag = np.zeros(n, dtype=np.int32)
            i32 = C.POINTER(C.c_int32)
            self.ctx.call("hpg_export_level", self.level, _lib.dptr(vals), cols.ctypes.data_as(i32),
                          nnz.ctypes.data_as(i32), diag.ctypes.data_as(i32))
            self._host = (vals, cols, nnz, diag)
        return self._host

    @property
    def values(self):
        v = self._export()[0]
        return v.astype(np.float32) if self.prec == _lib.F32 else v

    @property
    def col_idx(self):
        return self._export()[1]

    @property
    def row_nnz(self):
        return self._export()[2]

    @property
    def diag_pos(self):
        return self._export()[3]

    def diagonal(self):
        vals, _, _, diag = self._export()
        return vals[np.arange(self.n_rows), diag].astype(self.dtype)


def to_low_precision(A):
    """fp32 twin sharing the structure (ref: problem.py:165-175)."""
    return EllMatrix(A.ctx, A.level, _lib.F32)


@dataclass
class ProblemVectors:
    b: object
    x_exact: object
    x: object


def generate_rhs(A):
    """b = A 1 (row sums: 27 - nnz, exact), x_exact = 1, x = 0 (ref: problem.py:152-162)."""
    import torch
    dev = A.ctx.device
    ones = torch.ones(A.n_cols_extended, dtype=torch.float64, device=dev)
    b = torch.empty(A.n_rows, dtype=torch.float64, device=dev)
    A.ctx.call("hpg_spmv", A.level, _lib.F64, _lib.ptr(ones), _lib.ptr(b))
    # SpMV exchanged the halo of `ones` with the neighbours' ones: all exact.
    return ProblemVectors(b=b, x_exact=torch.ones(A.n_rows, dtype=torch.float64, device=dev),
                          x=torch.zeros(A.n_cols_extended, dtype=torch.float64, device=dev))


def structure_signature(A):
    """Hash of the structural arrays (ref: problem.py:178-186)."""
    import hashlib
    h = hashlib.sha256()
    vals, cols, nnz, diag = A._export()
    for arr in (cols, nnz, diag):
        h.update(np.ascontiguousarray(arr).tobytes())
    h.update(f"{A.n_rows}:{A.width}:{A.nnz_total}".encode())
    return h.hexdigest()


def host_level(local_dims, rank_coords=(0, 0, 0), proc_dims=(1, 1, 1)):
    """Reference-layout ELL of one rank-level computed by the library's host code.

    Same closed forms the device build kernel uses (csrc/hpg_geom.h); needs no GPU.
    Returns (values, col_idx, row_nnz, diag_pos, info).
    """
    n = int(np.prod(local_dims))
    vals = np.zeros((n, STENCIL_WIDTH))
    cols = np.zeros((n, STENCIL_WIDTH), dtype=np.int32)
    nnz = np.zeros(n, dtype=np.int32)
    diag = np.zeros(n, dtype=np.int32)
    info = np.zeros(14, dtype=np.int64)
    i32 = C.POINTER(C.c_int32)
    _lib.check(_lib.lib().hpg_host_level(
        _lib.ints(*local_dims), _lib.ints(*rank_coords), _lib.ints(*proc_dims),
        _lib.dptr(vals), cols.ctypes.data_as(i32), nnz.ctypes.data_as(i32),
        diag.ctypes.data_as(i32), info.ctypes.data_as(C.POINTER(C.c_int64)), 14))
    meta = {"n": int(info[0]), "n_ext": int(info[1]), "nnz": int(info[2]),
            "ncolors": int(info[3]), "color_offsets": info[4:4 + int(info[3]) + 1].copy(),
            "halo": int(info[13])}
    return vals, cols, nnz, diag, meta
