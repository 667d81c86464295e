"""HPG-MxP accounting: frozen flop/byte model, penalty, report (ref: metrics.py:1-161).

The model is the reference's, formula for formula (ref: metrics.py:37-77):
operations of every precision count equally, bytes move values at their
width and indices at 4 B, each touched once per kernel.  ``Tally`` keeps the
per-motif flops/bytes on the host and takes its seconds from CUDA events
recorded inside libhpgmxp around each motif (csrc/hpg_capi.cu ``Timed``)
instead of host perf_counter brackets.
"""

from __future__ import annotations

import json
import time
from contextlib import contextmanager

import numpy as np

MOTIFS = ("GS", "SpMV", "Ortho", "Restriction", "Prolongation", "Vector ops")


def _flops(kernel, n=0, k=0, nnz=0, n_c=0):
    table = {
        "spmv": 2 * nnz, "gs_sweep": 2 * nnz, "dot": 2 * n, "norm": 2 * n, "scale": n,
        "vsub": n, "vadd": n, "waxpby": 3 * n, "cgs2": 8 * n * k + 2 * n,
        "gemv_update": 2 * n * k, "restrict_fused": 2 * nnz + n_c, "restrict_inject": 0,
        "prolong_add": n_c,
    }
    return table[kernel]


def _bytes(kernel, w, n=0, k=0, nnz=0, n_c=0):
    table = {
        "spmv": nnz * (w + 4) + 2 * n * w, "gs_sweep": nnz * (w + 4) + 3 * n * w,
        "dot": 2 * n * w, "norm": n * w, "scale": 2 * n * w, "vsub": 3 * n * w,
        "vadd": 3 * n * w, "waxpby": 3 * n * w, "cgs2": 4 * n * k * w + 4 * n * w,
        "gemv_update": (n * k + 2 * n) * w, "restrict_fused": nnz * (2 * w + 4) + 2 * n_c * w,
        "restrict_inject": 2 * n_c * w, "prolong_add": 3 * n_c * w,
    }
    return table[kernel]


_MOTIF = {"spmv": "SpMV", "gs_sweep": "GS", "dot": "Vector ops", "norm": "Vector ops",
          "scale": "Vector ops", "vsub": "Vector ops", "vadd": "Vector ops",
          "waxpby": "Vector ops", "cgs2": "Ortho", "gemv_update": "Ortho",
          "restrict_fused": "Restriction", "restrict_inject": "Restriction",
          "prolong_add": "Prolongation"}

_SIZES = {"spmv": ("nnz", "n"), "gs_sweep": ("nnz", "n"), "dot": ("n",), "norm": ("n",),
          "scale": ("n",), "vsub": ("n",), "vadd": ("n",), "waxpby": ("n",),
          "cgs2": ("n", "k"), "gemv_update": ("n", "k"), "restrict_fused": ("nnz", "n_c"),
          "restrict_inject": ("n_c",), "prolong_add": ("n_c",)}


def _check(kernel, sizes):
    if kernel not in _MOTIF:
        raise ValueError(f"unknown kernel: {kernel!r}")
    if set(sizes) != set(_SIZES[kernel]):
        raise TypeError(f"{kernel} takes sizes {_SIZES[kernel]}, got {tuple(sizes)}")


def count_flops(kernel, **sizes):
    """Frozen operation count for one kernel invocation (ref: metrics.py:80-84)."""
    _check(kernel, sizes)
    return int(_flops(kernel, **sizes))


def count_bytes(kernel, value_width, **sizes):
    """Modelled traffic for one kernel invocation (ref: metrics.py:87-91)."""
    _check(kernel, sizes)
    return int(_bytes(kernel, value_width, **sizes))


def kernel_motif(kernel):
    return _MOTIF[kernel]


def penalty_factor(n_d, n_ir):
    """min(1, n_d / n_ir) (ref: metrics.py:98-102)."""
    if n_d < 1 or n_ir < 1:
        raise ValueError(f"iteration counts must be >= 1, got ({n_d}, {n_ir})")
    return min(1.0, n_d / n_ir)


def gflops(flops, seconds):
    if seconds <= 0:
        raise ValueError(f"need positive seconds, got {seconds}")
    return flops / seconds / 1e9


class Tally:
    """Per-rank flops / model bytes / seconds per motif (ref: metrics.py:111-143).

    Beside the reference's model it keeps, per motif, the flops the kernels
    actually EXECUTE (``exec_flops``: lower than the model only for the optional
    strictly-lower zero-guess sweep) and the bytes they actually MOVE
    (``moved_bytes``: the model minus the 4-B column indices that implicit-index
    rows compute instead of loading, and the lower part only for that sweep).
    """

    def __init__(self):
        self.flops = {m: 0 for m in MOTIFS}
        self.bytes = {m: 0 for m in MOTIFS}
        self.seconds = {m: 0.0 for m in MOTIFS}
        self.exec_flops = {m: 0 for m in MOTIFS}
        self.moved_bytes = {m: 0 for m in MOTIFS}
        # subsets of GS timed alone for the bench roofline: level-0 full sweeps
        # (k_gs_pass, model bytes) and level-0 zero-initial-guess sweeps
        # (k_gs_lower, the bytes that kernel streams)
        self.gs_level0_seconds = 0.0
        self.gs_level0_bytes = 0
        self.gs_level0_sweeps = 0
        self.gs_level0z_seconds = 0.0
        self.gs_level0z_bytes = 0
        self.gs_level0z_sweeps = 0

    def add(self, kernel, dtype, motif=None, implicit_nnz=0, exec_flops=None, moved=None, **sizes):
        """``implicit_nnz``: nonzeros whose column the kernel computes (no 4-B index
        load); ``exec_flops`` / ``moved``: override both extra counts outright."""
        bucket = motif or kernel_motif(kernel)
        f = count_flops(kernel, **sizes)
        b = count_bytes(kernel, np.dtype(dtype).itemsize, **sizes)
        self.flops[bucket] += f
        self.bytes[bucket] += b
        self.exec_flops[bucket] += f if exec_flops is None else int(exec_flops)
        self.moved_bytes[bucket] += (b - 4 * int(implicit_nnz)) if moved is None else int(moved)

    @contextmanager
    def timed(self, motif):
        """Host wall-clock bracket (only for host-side work; device motifs use events)."""
        t0 = time.perf_counter()
        try:
            yield
        finally:
            self.seconds[motif] += time.perf_counter() - t0

    def absorb_device_seconds(self, ctx):
        """Add the library's per-motif CUDA-event seconds and reset them."""
        sec = ctx.timers(2)
        for m, s in zip(MOTIFS, sec):
            self.seconds[m] += float(s)
        self.gs_level0_seconds += float(sec[6])
        self.gs_level0z_seconds += float(sec[7])

    def total_flops(self):
        return sum(self.flops.values())

    def total_bytes(self):
        return sum(self.bytes.values())

    def total_exec_flops(self):
        return sum(self.exec_flops.values())

    def total_moved_bytes(self):
        return sum(self.moved_bytes.values())

    def reset(self):
        for m in MOTIFS:
            self.flops[m] = 0
            self.bytes[m] = 0
            self.seconds[m] = 0.0
            self.exec_flops[m] = 0
            self.moved_bytes[m] = 0
        self.gs_level0_seconds = 0.0
        self.gs_level0_bytes = 0
        self.gs_level0_sweeps = 0
        self.gs_level0z_seconds = 0.0
        self.gs_level0z_bytes = 0
        self.gs_level0z_sweeps = 0


def sum_motif_dicts(dicts):
    out = {m: 0 for m in MOTIFS}
    for d in dicts:
        for m in MOTIFS:
            out[m] += d[m]
    return out


def emit_report(report):
    """Serialise the report (stable field names are the contract; ref: metrics.py:155-157)."""
    return json.dumps(report, indent=2)


def parse_report(text):
    return json.loads(text)
