"""Forward multicolor Gauss-Seidel (ref: smoother.py:1-115).

One sweep = one exchange of z's halo (block-Jacobi between ranks, skipped
when ``z_is_zero``) followed by one kernel per color block in order
(csrc/hpg_kernels.cuh k_gs_pass).  Bitwise identical to the reference sweep:
same slot order, separate IEEE mul/add, IEEE divide by a_ii.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib


class SingularDiagonal(Exception):
    """A zero diagonal entry reached the smoother (ref: smoother.py:23-24)."""


@dataclass
class SmootherWorkspace:
    """Sweep counts nu1 / nu2 / nu_c (ref: smoother.py:27-37)."""

    nu1: int = 1
    nu2: int = 1
    nu_c: int = 1

    def __post_init__(self):
        if min(self.nu1, self.nu2, self.nu_c) < 1:
            raise ValueError("sweep counts must all be >= 1")


def forward_gs_sweep(A, r, z, coloring=None, plan=None, world=None, rank=0,
                     z_is_zero=False, overlap=True, tally=None):
    """z <- one forward GS sweep of A z = r (z carries the halo tail; in place).

    ``coloring``/``plan``/``world``/``overlap`` are accepted for signature
    parity (ref: smoother.py:78-79); the device level already knows its
    color blocks and halo plan.
    """
    rd, _ = _lib.on_device(r, A.torch_dtype, A.ctx.device)
    zd, zh = _lib.on_device(z, A.torch_dtype, A.ctx.device)
    if zh is not None and zh.dtype != A.dtype:
        raise TypeError(f"GS sweep operands must be {A.dtype}")
    r, z = rd, zd
    if z.dtype != A.torch_dtype or r.dtype != A.torch_dtype:
        raise TypeError(f"GS sweep operands must be {A.torch_dtype}")
    if coloring is not None:  # the sweep runs over the level's own colour blocks: they must agree
        info = A.ctx.level_info(A.level)
        offs = [info[f"off{k}"] for k in range(info["ncolors"] + 1)]
        if int(coloring.num_colors) != info["ncolors"] or \
                [int(o) for o in coloring.color_offsets] != offs[:int(coloring.num_colors) + 1]:
            raise ValueError("coloring does not match the operand's colour blocks")
    A.ctx.call("hpg_gs_sweep", A.level, A.prec, _lib.ptr(r), _lib.ptr(z), int(bool(z_is_zero)))
    _lib.back_to_host(z, zh)
    if tally is not None:
        zs = None
        if z_is_zero and A.ctx.option("lower"):
            from .multigrid import zero_sweep_counts

            class _H:  # zero_sweep_counts needs only the context
                ctx = A.ctx
            zs = zero_sweep_counts(_H, A.level, A.dtype.itemsize)
        if zs is not None:
            tally.add("gs_sweep", A.dtype, nnz=A.nnz_total, n=A.n_rows, exec_flops=zs[0], moved=zs[1])
        else:
            tally.add("gs_sweep", A.dtype, nnz=A.nnz_total, n=A.n_rows, implicit_nnz=A.implicit_nnz)
