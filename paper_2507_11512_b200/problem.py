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
    def local_dims(self):
        """The rank-local box of this operand (what ``coloring.color`` reads)."""
        return self.domain.local_dims

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
        # one host export per (context, level), shared by the fp64 / fp32 twins
        # (the reference's low-precision copy shares its structure arrays)
        cache = self.ctx.__dict__.setdefault("_host_export", {})
        if self._host is None and self.level in cache:
            self._host = cache[self.level]
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
            cache[self.level] = self._host
        return self._host

    def global_rows(self):
        """Global id of every row in this operand's row order."""
        d = self.domain
        perm = self.row_perm()
        lx, ly, _ = d.local_dims
        x, y, z = perm % lx, (perm // lx) % ly, perm // (lx * ly)
        return (d.ox + x) + d.gnx * ((d.oy + y) + d.gny * (d.oz + z))

    def row_perm(self):
        """Natural (pre-reorder) index of every row: the level's colouring."""
        if getattr(self, "natural", False):
            return np.arange(self.n_rows, dtype=np.int64)
        col = getattr(self, "coloring", None)
        if col is None:
            from .coloring import greedy_coloring
            col = greedy_coloring(*self.domain.local_dims)
        return np.asarray(col.perm, dtype=np.int64)

    @property
    def col_global(self):
        """Global column id of every entry, -1 for padding (ref: problem.py:31-57):
        slot k of a row is its k-th in-domain neighbour in ascending global id."""
        cache = self.ctx.__dict__.setdefault("_col_global", {})
        if self.level not in cache:
            d = self.domain
            g = self.global_rows()
            gx, gy, gz = g % d.gnx, (g // d.gnx) % d.gny, g // (d.gnx * d.gny)
            cols = np.full((len(g), STENCIL_WIDTH), -1, dtype=np.int64)
            k = np.zeros(len(g), dtype=np.int64)
            rows = np.arange(len(g))
            for dz in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    for dx in (-1, 0, 1):
                        ax, ay, az = gx + dx, gy + dy, gz + dz
                        ok = (ax >= 0) & (ax < d.gnx) & (ay >= 0) & (ay < d.gny) & (az >= 0) & (az < d.gnz)
                        cols[rows[ok], k[ok]] = (ax + d.gnx * (ay + d.gny * az))[ok]
                        k += ok
            cache[self.level] = cols
        return cache[self.level]

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


def generate_matrix(domain, world=None):
    """The rank-local 27-point operand of ``domain`` in NATURAL row order
    (ref: problem.py:88-142), assembled on the device: a one-level context whose
    row order is the identity permutation (one colour block).  Compact rows,
    ascending global columns, padding column 0 / value 0, 26 / -1 values -- the
    exported ``values`` / ``col_idx`` / ``row_nnz`` / ``diag_pos`` are the
    reference's, except that off-rank columns already carry their halo slots
    (the device builds the halo plan with the level; ``build_halo_plan`` then
    hands it out).  Several ranks: pass the job's ``world`` (an extension: the
    device context needs its communicator at creation)."""
    from .device import Context
    if domain.npx * domain.npy * domain.npz > 1 and world is None:
        raise ValueError("a multi-rank domain needs world= (the device context's communicator)")
    ctx = Context(domain, 1, world=world)
    n = domain.n_rows
    offs = np.array([0, n], dtype=np.int64)
    perm = np.arange(n, dtype=np.int64)
    i64 = C.POINTER(C.c_int64)
    ctx.call("hpg_set_coloring", 0, 1, offs.ctypes.data_as(i64), perm.ctypes.data_as(i64))
    A = EllMatrix(ctx, 0, _lib.F64)
    A.domain = domain
    A.world = world
    A.natural = True
    return A


def matrix_market_lines(A, global_rows):
    """'row col value' lines (1-based global ids) of A's rows in A's row order
    (ref: problem.py:216-223)."""
    vals, nnz, cols = A.values, A.row_nnz, A.col_global
    g = np.asarray(global_rows, dtype=np.int64)
    out = []
    for i in range(len(g)):
        r = int(g[i]) + 1
        for s in range(int(nnz[i])):
            v = float(vals[i, s])
            out.append(f"{r} {int(cols[i, s]) + 1} {int(v) if v.is_integer() else repr(v)}\n")
    return out


def write_matrix_market(path, A, global_rows, n_global):
    """Local rows as MatrixMarket coordinate triplets, global ids (ref: problem.py:193-213)."""
    lines = matrix_market_lines(A, global_rows)
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{n_global} {n_global} {A.nnz_total}\n")
        f.writelines(lines)


def to_low_precision(A):
    """fp32 twin sharing the structure (ref: problem.py:165-175)."""
    lo = EllMatrix(A.ctx, A.level, _lib.F32)
    for k in ("domain", "world", "natural"):
        if hasattr(A, k):
            setattr(lo, k, getattr(A, k))
    return lo


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
