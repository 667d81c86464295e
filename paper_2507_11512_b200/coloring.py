"""Multicolor ordering of a rank-level (ref: coloring.py:16-123).

On the structured 27-point lattice the reference's greedy first-fit coloring
(ref: coloring.py:49-55) is the parity pattern of the local coordinates over
the axes with extent >= 2, and its (color, natural index) permutation
(ref: coloring.py:78-80) is closed form.  The device never materialises it:
the build kernels evaluate csrc/hpg_geom.h iperm() per row.  This module
produces the same ``Coloring`` record on the host for callers and tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Coloring:
    color: np.ndarray          # color per natural (pre-reorder) row
    num_colors: int
    color_offsets: np.ndarray  # block start per color after reordering
    perm: np.ndarray           # new row -> natural row
    iperm: np.ndarray          # natural row -> new row


def greedy_coloring(lx, ly, lz):
    dims = (lx, ly, lz)
    n = lx * ly * lz
    bits = {}
    for a in range(3):
        if dims[a] >= 2:
            bits[a] = len(bits)
    nat = np.arange(n, dtype=np.int64)
    coords = (nat % lx, (nat // lx) % ly, nat // (lx * ly))
    color = np.zeros(n, dtype=np.int32)
    for a, b in bits.items():
        color |= ((coords[a] & 1) << b).astype(np.int32)
    num_colors = (1 << len(bits)) if n else 0
    counts = np.bincount(color, minlength=num_colors)
    offsets = np.zeros(num_colors + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    perm = np.lexsort((nat, color))
    iperm = np.empty_like(perm)
    iperm[perm] = nat
    return Coloring(color=color, num_colors=num_colors, color_offsets=offsets, perm=perm,
                    iperm=iperm)


def _local_neighbours(lx, ly, lz, rows):
    """[len(rows), 26] natural indices of the in-box 27-point neighbours (-1: none), ascending."""
    x, y, z = rows % lx, (rows // lx) % ly, rows // (lx * ly)
    out = np.full((len(rows), 26), -1, dtype=np.int64)
    s = 0
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                if dx == dy == dz == 0:
                    continue
                ax, ay, az = x + dx, y + dy, z + dz
                ok = (ax >= 0) & (ax < lx) & (ay >= 0) & (ay < ly) & (az >= 0) & (az < lz)
                out[ok, s] = (ax + lx * (ay + ly * az))[ok]
                s += 1
    return out


def jpl_coloring_device(lx, ly, lz, seed=0, device=None):
    """JPL on the GPU (csrc/hpg_jpl.cuh, ``hpg_jpl_color``): the reference's
    rounds with its exact random stream -- numpy's default_rng(seed) PCG64 state
    handed to the device, each draw reached by jump-ahead.  Bit-identical to
    ``jpl_coloring`` and the reference (ref: coloring.py:56-70)."""
    import ctypes as C
    from . import _lib
    if device is None:
        import torch
        device = torch.cuda.current_device()
    st = np.random.default_rng(seed).bit_generator.state["state"]
    m64 = (1 << 64) - 1
    state = (C.c_uint64 * 2)(st["state"] & m64, st["state"] >> 64)
    inc = (C.c_uint64 * 2)(st["inc"] & m64, st["inc"] >> 64)
    n = lx * ly * lz
    colors = np.empty(n, dtype=np.int32)
    rounds = C.c_int()
    _lib.check(_lib.lib().hpg_jpl_color(int(device), lx, ly, lz, state, inc,
                                        colors.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(rounds)))
    return _coloring_from_colors(colors)


def _coloring_from_colors(colors):
    n = len(colors)
    num_colors = int(colors.max()) + 1 if n else 0
    counts = np.bincount(colors, minlength=num_colors)
    offsets = np.zeros(num_colors + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    perm = np.argsort(colors, kind="stable").astype(np.int64)  # (colour, natural index)
    iperm = np.empty_like(perm)
    iperm[perm] = np.arange(n, dtype=np.int64)
    return Coloring(color=colors, num_colors=num_colors, color_offsets=offsets, perm=perm, iperm=iperm)


def jpl_coloring(lx, ly, lz, seed=0, chunk=1 << 20):
    """Jones-Plassmann-Luby coloring, vectorised, identical to the reference's
    (ref: coloring.py:56-70): each round draws rng.random(n); a remaining row is
    selected when (w_i, i) beats (w_j, j) of every remaining local neighbour; each
    selected row takes the smallest color its already colored neighbours lack.
    Selected rows are independent, so they can be colored all at once."""
    n = lx * ly * lz
    colors = np.full(n, -1, dtype=np.int32)
    remaining = np.ones(n, dtype=bool)
    rng = np.random.default_rng(seed)
    while remaining.any():
        w = rng.random(n)
        sel = np.zeros(n, dtype=bool)
        for a in range(0, n, chunk):
            rows = np.arange(a, min(n, a + chunk), dtype=np.int64)
            nb = _local_neighbours(lx, ly, lz, rows)
            valid = nb >= 0
            nbc = np.where(valid, nb, 0)
            live = valid & remaining[nbc]
            wi, wj = w[rows][:, None], w[nbc]
            beats = (wi > wj) | ((wi == wj) & (rows[:, None] > nbc))
            sel[rows] = remaining[rows] & np.all(beats | ~live, axis=1)
        idx = np.flatnonzero(sel)
        for a in range(0, len(idx), chunk):
            rows = idx[a:a + chunk]
            nb = _local_neighbours(lx, ly, lz, rows)
            cn = np.where(nb >= 0, colors[np.where(nb >= 0, nb, 0)], -1)
            used = np.zeros(len(rows), dtype=np.int64)
            for s in range(26):
                c = cn[:, s]
                used |= np.where(c >= 0, np.left_shift(1, np.maximum(c, 0)), 0)
            free = ~used
            colors[rows] = (np.log2((free & -free).astype(np.float64))).astype(np.int32)
        remaining &= ~sel
    num_colors = int(colors.max()) + 1 if n else 0
    counts = np.bincount(colors, minlength=num_colors)
    offsets = np.zeros(num_colors + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    nat = np.arange(n, dtype=np.int64)
    perm = np.lexsort((nat, colors))
    iperm = np.empty_like(perm)
    iperm[perm] = nat
    return Coloring(color=colors, num_colors=num_colors, color_offsets=offsets, perm=perm, iperm=iperm)


def color(A_or_dims, strategy="greedy", seed=0):
    """Coloring of a level given its local dims (or a domain with ``local_dims``)
    (ref: coloring.py:36-82)."""
    dims = getattr(A_or_dims, "local_dims", A_or_dims)
    if strategy == "greedy":
        return greedy_coloring(*dims)
    if strategy == "jpl":
        # on the GPU when there is one (setup at 256^3 in well under a second); the
        # vectorised host restatement otherwise (CPU-only tooling and tests)
        try:
            import torch
            if torch.cuda.is_available():
                return jpl_coloring_device(*dims, seed=seed)
        except ImportError:
            pass
        return jpl_coloring(*dims, seed=seed)
    raise ValueError(f"unknown coloring strategy: {strategy!r}")


def identity_coloring(n):
    """One colour, natural order (ref: coloring.py:84-88)."""
    return Coloring(color=np.zeros(n, dtype=np.int32), num_colors=1,
                    color_offsets=np.array([0, n], dtype=np.int64),
                    perm=np.arange(n), iperm=np.arange(n))


def check_coloring(A, coloring):
    """True iff no two locally coupled rows share a colour (ref: coloring.py:91-98).
    ``A`` (or a domain / local dims) gives the local box; rows in natural order."""
    dims = getattr(A, "local_dims", A)
    lx, ly, lz = dims
    n = lx * ly * lz
    rows = np.arange(n, dtype=np.int64)
    nb = _local_neighbours(lx, ly, lz, rows)
    col = np.asarray(coloring.color)
    ok = nb >= 0
    return not np.any(ok & (col[np.where(ok, nb, 0)] == col[:, None]))


def permute_system(A, vectors, coloring):
    """The symmetric reordering P A P^T and P v (ref: coloring.py:101-123).

    On the device this is a new level in the colouring's row order: the greedy
    colouring keeps the closed-form layout (implicit-index rows, dataflow
    sweeps), any other colouring is installed as an explicit permutation.
    Returns (operand, permuted copies of ``vectors``)."""
    import ctypes as C
    from . import _lib
    from .device import Context
    from .problem import EllMatrix
    dom = A.domain
    world = getattr(A, "world", None)
    ctx = Context(dom, 1, world=world)
    greedy = greedy_coloring(*dom.local_dims)
    if not (coloring.num_colors == greedy.num_colors and np.array_equal(coloring.perm, greedy.perm)):
        offs = np.ascontiguousarray(coloring.color_offsets, dtype=np.int64)
        perm = np.ascontiguousarray(coloring.perm, dtype=np.int64)
        i64 = C.POINTER(C.c_int64)
        ctx.call("hpg_set_coloring", 0, int(coloring.num_colors), offs.ctypes.data_as(i64),
                 perm.ctypes.data_as(i64))
    out = EllMatrix(ctx, 0, _lib.F64)
    out.domain, out.world, out.coloring = dom, world, coloring
    vecs = []
    for v in vectors:
        if isinstance(v, np.ndarray):
            vecs.append(v[coloring.perm].copy())
        else:
            import torch
            vecs.append(v[torch.as_tensor(coloring.perm, device=v.device)].clone())
    return out, vecs
