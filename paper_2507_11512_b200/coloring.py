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


def color(A_or_dims, strategy="greedy", seed=0):
    """Coloring of a level given its local dims (or a domain with ``local_dims``)."""
    if strategy != "greedy":
        raise NotImplementedError(
            f"coloring strategy {strategy!r}: only 'greedy' is built for the device path "
            "(JPL is SURVEY.md 8(f) F4)")
    dims = getattr(A_or_dims, "local_dims", A_or_dims)
    return greedy_coloring(*dims)
