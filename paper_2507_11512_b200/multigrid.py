"""Geometric multigrid on the device (ref: multigrid.py:1-172).

``build_hierarchy`` creates one libhpgmxp context that generates every level
in HBM (csrc/hpg_capi.cu build_level): permuted ELL in fp64 and fp32,
halo plans, injection maps and V-cycle workspaces.  ``MgHierarchy.apply``
runs the whole V-cycle inside the library (one C call, no host round trips);
``mg_vcycle`` is the same algorithm spelled out over the per-kernel entry
points, kept for API parity and as a differential test of ``apply``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .coloring import color as color_rows
from .comm import HaloPlan
from .device import Context
from .problem import EllMatrix
from .smoother import SmootherWorkspace, forward_gs_sweep


@dataclass
class MgLevel:
    domain: object
    A_hi: object
    A_lo: object
    coloring: object = None
    plan: object = None
    f2c: object = None
    z_hi: object = None
    z_lo: object = None
    r_hi: object = None
    r_lo: object = None


@dataclass
class MgHierarchy:
    levels: list
    sweeps: SmootherWorkspace
    world: object = None
    rank: int = 0
    ctx: object = field(default=None, repr=False)

    def apply(self, r, tally=None, out=None, count=True):
        """One V-cycle from the finest level; precision follows r's dtype (ref: multigrid.py:49-51).

        Returns the level-0 workspace view (or ``out[:n]`` when given, out having
        the halo tail) -- consume it before the next call, like the reference.
        """
        import torch
        lv = self.levels[0]
        if isinstance(r, np.ndarray):  # host array: V-cycle on the device, copy of z back
            lo = r.dtype == np.float32
            rd, _ = _lib.on_device(r, torch.float32 if lo else torch.float64, self.ctx.device)
            return self.apply(rd, tally, None, count).cpu().numpy()
        lo = r.dtype == torch.float32
        A = lv.A_lo if lo else lv.A_hi
        z = out if out is not None else (lv.z_lo if lo else lv.z_hi)
        # a tallied V-cycle outside a solve times its own motifs (CUDA events)
        own = tally is not None and count and not getattr(self.ctx, "timing", False)
        if own:
            self.ctx.timers(1)
        self.ctx.call("hpg_vcycle", A.prec, _lib.ptr(r), _lib.ptr(z))
        if tally is not None and count:
            count_vcycle(self, tally, A.dtype)
        if own:
            tally.absorb_device_seconds(self.ctx)
            self.ctx.timers(0)
        return z[:A.n_rows]

    def preconditioner(self, tally=None):
        """Callable precond(r, out=None) for gmres_solve (writes into out when given)."""
        hier = self
        last = {}

        def precond(r, out=None, count=True):
            last["dtype"] = np.float32 if r.dtype.itemsize == 4 else np.float64
            return hier.apply(r, tally, out, count)

        def account():
            """Tally one V-cycle (for applications issued with count=False)."""
            if tally is not None:
                count_vcycle(hier, tally, last.get("dtype", np.float64))

        precond.accepts_out = True
        precond.account = account
        return precond

    def close(self):
        if self.ctx is not None:
            self.ctx.close()
            self.ctx = None


def count_vcycle(h, tally, dtype):
    """Flop/byte accounting of one V-cycle, call by call as the reference tallies it
    (model), plus the executed flops and moved bytes of the kernels that ran."""
    nl = len(h.levels)
    sw = h.sweeps
    w = np.dtype(dtype).itemsize
    for lev in range(nl):
        A = h.levels[lev].A_hi
        last = lev == nl - 1
        sweeps = sw.nu_c if last else sw.nu1 + sw.nu2
        for k in range(sweeps):
            zs = zero_sweep_counts(h, lev, w) if k == 0 else None
            if zs is not None:  # strictly-lower zero-guess sweep (option "lower")
                tally.add("gs_sweep", dtype, nnz=A.nnz_total, n=A.n_rows, exec_flops=zs[0], moved=zs[1])
            else:
                tally.add("gs_sweep", dtype, nnz=A.nnz_total, n=A.n_rows, implicit_nnz=A.implicit_nnz)
            if lev == 0 and hasattr(tally, "gs_level0_bytes"):
                if zs is not None:
                    tally.gs_level0z_bytes += zs[1]
                    tally.gs_level0z_sweeps += 1
                else:
                    from .metrics import count_bytes
                    tally.gs_level0_bytes += count_bytes("gs_sweep", w, nnz=A.nnz_total, n=A.n_rows)
                    tally.gs_level0_sweeps += 1
        if not last:
            nxt = h.levels[lev + 1]
            tally.add("restrict_fused", dtype, nnz=nxt.inject_nnz, n_c=nxt.A_hi.n_rows,
                      implicit_nnz=restrict_implicit_nnz(h, lev))
            tally.add("prolong_add", dtype, n_c=nxt.A_hi.n_rows)


def zero_sweep_counts(h, lev, w):
    """(executed flops, moved bytes) of a zero-initial-guess sweep at ``lev`` when it
    runs the strictly-lower kernel (csrc/hpg_lower.cuh), else None (the sweep runs
    the full color-pass kernel and forms every product like the reference, the
    ones against z = 0 included)."""
    if h.ctx is None or not h.ctx.option("lower"):
        return None
    info = h.ctx.level_info(lev)
    n, slots = info["n"], info["zero_sweep_slots"]
    if slots >= 27 * n:
        return None
    idx_rows = n - info["stencil_rows"] if info["stencil_lower"] and h.ctx.option("stencil") else n
    # W_c products + (r - sum) / a_ii per row; lower values (+ indices of indexed
    # rows, pro rata), a_ii, r, z written, z gathered once
    return 2 * slots + 2 * n, slots * w + 4 * slots * idx_rows // max(n, 1) + 4 * n * w


def restrict_implicit_nnz(h, lev):
    """Nonzeros of the injected fine rows on the implicit-index path (pro rata)."""
    A = h.levels[lev].A_hi
    nxt = h.levels[lev + 1]
    if A.n_rows == 0:
        return 0
    return nxt.inject_nnz * (A.implicit_nnz // 27) // A.n_rows


def zero_sweep_bytes(h, w):
    """Bytes one level-0 zero-initial-guess sweep streams (see zero_sweep_counts)."""
    zs = zero_sweep_counts(h, 0, w)
    return zs[1] if zs is not None else full_sweep_moved_bytes(h, w)


def full_sweep_moved_bytes(h, w):
    """Bytes one level-0 full sweep (8 color passes) streams: every value, the column
    indices of the rows off the implicit-index path, r, z gathered once, z written."""
    info = h.ctx.level_info(0)
    n = info["n"]
    idx_rows = n - info["stencil_rows"] if h.ctx.option("stencil") else n
    return info["nnz"] * w + 27 * 4 * idx_rows + 3 * n * w


def _inject_nnz(domain):
    """nnz of the fine rows at injection points (even local coords) -- closed form."""
    tot = 1
    for l, o, g in ((domain.lnx, domain.ox, domain.gnx), (domain.lny, domain.oy, domain.gny),
                    (domain.lnz, domain.oz, domain.gnz)):
        s = 0
        for x in range(0, l, 2):
            s += sum(1 for d in (-1, 0, 1) if 0 <= o + x + d < g)
        tot *= s
    return tot


def build_hierarchy(domain, levels, world=None, rank=0, strategy="greedy", seed=0, sweeps=None):
    """Generate, color, reorder and plan every level on the device (ref: multigrid.py:54-84)."""
    import torch
    if levels < 1:
        raise ValueError("need at least one level")
    if strategy not in ("greedy", "jpl"):
        raise ValueError(f"unknown coloring strategy: {strategy!r}")
    sweeps = sweeps or SmootherWorkspace()
    doms = [domain]
    for _ in range(levels - 1):
        doms.append(doms[-1].coarsen())  # CoarseningError, like the reference
    ctx = Context(domain, levels, sweeps.nu1, sweeps.nu2, sweeps.nu_c, world)
    colorings = [None] * levels
    if strategy == "jpl":
        # host JPL per level (same RNG stream as the reference), then the device
        # rebuilds each level in that order (ref: multigrid.py:66-70)
        import ctypes as C
        for lev, dom in enumerate(doms):
            col = color_rows(dom, "jpl", seed)
            colorings[lev] = col
            offs = np.ascontiguousarray(col.color_offsets, dtype=np.int64)
            perm = np.ascontiguousarray(col.perm, dtype=np.int64)
            i64 = C.POINTER(C.c_int64)
            ctx.call("hpg_set_coloring", lev, col.num_colors, offs.ctypes.data_as(i64),
                     perm.ctypes.data_as(i64))
    out = []
    for lev, dom in enumerate(doms):
        A = EllMatrix(ctx, lev, _lib.F64)
        A_lo = EllMatrix(ctx, lev, _lib.F32)
        A.domain = A_lo.domain = dom
        A.coloring = A_lo.coloring = colorings[lev]  # None: the greedy closed form
        lv = MgLevel(domain=dom, A_hi=A, A_lo=A_lo, coloring=colorings[lev])
        lv.plan = HaloPlan(ctx, lev, dom) if world is not None else None
        ne, n = A.n_cols_extended, A.n_rows
        dev = ctx.device
        lv.z_hi = torch.zeros(ne, dtype=torch.float64, device=dev)
        lv.z_lo = torch.zeros(ne, dtype=torch.float32, device=dev)
        lv.r_hi = torch.zeros(n, dtype=torch.float64, device=dev)
        lv.r_lo = torch.zeros(n, dtype=torch.float32, device=dev)
        if lev > 0:
            lv.inject_nnz = _inject_nnz(doms[lev - 1])
        out.append(lv)
    h = MgHierarchy(levels=out, sweeps=sweeps, world=world, rank=rank, ctx=ctx)
    for lev in range(1, levels):
        out[lev].f2c = Injection(h, lev)
    return h


def level_coloring(lv):
    if lv.coloring is None:
        lv.coloring = color_rows(lv.domain)
    return lv.coloring


def injection_map(h, level):
    """f2c of ``level`` (>= 1) into its parent, as host int64 (ref: multigrid.py:87-99)."""
    import ctypes as C
    n = h.levels[level].A_hi.n_rows
    f2c = np.zeros(n, dtype=np.int64)
    h.ctx.call("hpg_export_f2c", level, f2c.ctypes.data_as(C.POINTER(C.c_int64)))
    return f2c


class Injection:
    """A coarse level's injection map f2c (coarse row i <- fine row f2c[i]),
    held on the device by the hierarchy (ref: multigrid.py:87-99 _injection_map).

    What ``MgLevel.f2c`` holds: usable wherever the reference passes f2c
    (``prolong_add``, ``restrict_inject``, ``fused_residual_restrict``) and
    array-like on the host (``np.asarray(lv.f2c)``, ``len``, indexing)."""

    def __init__(self, hier, level):
        self._hier = hier
        self.level = level            # the coarse level this map feeds
        self.fine_level = level - 1
        self._host = None
        self._dev = None

    @property
    def ctx(self):
        return self._hier.ctx

    def host(self):
        if self._host is None:
            self._host = injection_map(self._hier, self.level)
        return self._host

    def device(self):
        if self._dev is None:
            import torch
            self._dev = torch.from_numpy(self.host()).to(self.ctx.device)
        return self._dev

    def __array__(self, dtype=None, copy=None):
        a = self.host()
        return a.astype(dtype) if dtype is not None else a

    def __len__(self):
        return int(self._hier.levels[self.level].A_hi.n_rows)

    def __getitem__(self, k):
        return self.host()[k]


def restrict_inject(v_f, f2c):
    """Coarse vector of the fine values at injection points (ref: multigrid.py:102-104)."""
    if isinstance(v_f, np.ndarray):
        return v_f[np.asarray(f2c)].copy()
    idx = f2c.device() if isinstance(f2c, Injection) else f2c
    return v_f[idx].clone()


def fused_residual_restrict(A_f, b_f, x_f, f2c=None, out=None, tally=None, n_c=None):
    """r_c = (b_f - A_f x_f) at the injected rows; x_f's halo must be fresh (ref: multigrid.py:107-128).

    ``A_f`` is the fine level's operand; the injection map is the coarse level's,
    held on the device (``f2c``, the coarse level's ``MgLevel.f2c``, names it and
    must belong to the same hierarchy).
    """
    if isinstance(f2c, Injection) and (f2c.ctx is not A_f.ctx or f2c.fine_level != A_f.level):
        raise ValueError("f2c is not the injection map below this operand's level")
    import torch
    info = A_f.ctx.level_info(A_f.level + 1)
    bd, _ = _lib.on_device(b_f, A_f.torch_dtype, A_f.ctx.device)
    xd, _ = _lib.on_device(x_f, A_f.torch_dtype, A_f.ctx.device)
    outd, outh = _lib.on_device(out, A_f.torch_dtype, A_f.ctx.device) if out is not None else (None, None)
    if outd is None:
        outd = torch.empty(info["n"], dtype=A_f.torch_dtype, device=xd.device)
    A_f.ctx.call("hpg_restrict", A_f.level, A_f.prec, _lib.ptr(bd), _lib.ptr(xd), _lib.ptr(outd))
    if tally is not None:
        inj = _inject_nnz(A_f.domain)
        tally.add("restrict_fused", A_f.dtype, nnz=inj, n_c=info["n"],
                  implicit_nnz=inj * (A_f.implicit_nnz // 27) // max(A_f.n_rows, 1))
    if isinstance(x_f, np.ndarray):  # host arrays in, host result out
        if outh is not None:
            _lib.back_to_host(outd, outh)
            return outh
        return outd.cpu().numpy()
    return outd


def prolong_add(x_f, x_c, f2c, tally=None):
    """x_f[f2c] += x_c on the device, in place (ref: multigrid.py:131-137).

    ``f2c`` is the coarse level's injection map (``MgLevel.f2c``); it names the
    hierarchy and the level pair.  The precision follows the vectors'.
    """
    import torch
    if not isinstance(f2c, Injection):
        raise TypeError("f2c must be a level's injection map (MgLevel.f2c of a device hierarchy)")
    prec = _lib.F32 if x_f.dtype.itemsize == 4 else _lib.F64
    if x_c.dtype != x_f.dtype:
        raise TypeError("prolong_add operands must share one precision")
    tdt = torch.float32 if prec == _lib.F32 else torch.float64
    xf, xfh = _lib.on_device(x_f, tdt, f2c.ctx.device)
    xc, _ = _lib.on_device(x_c, tdt, f2c.ctx.device)
    f2c.ctx.call("hpg_prolong", f2c.fine_level, prec, _lib.ptr(xf), _lib.ptr(xc))
    _lib.back_to_host(xf, xfh)
    if tally is not None:
        tally.add("prolong_add", np.float32 if prec == _lib.F32 else np.float64, n_c=x_c.numel())


def mg_vcycle(h, level, r, tally=None):
    """The V-cycle over the per-kernel entry points (ref: multigrid.py:140-171)."""
    import torch
    lv = h.levels[level]
    lo = r.dtype == torch.float32
    A = lv.A_lo if lo else lv.A_hi
    z = lv.z_lo if lo else lv.z_hi
    sw = h.sweeps
    last = level == len(h.levels) - 1
    for s in range(sw.nu_c if last else sw.nu1):
        forward_gs_sweep(A, r, z, z_is_zero=(s == 0), tally=tally)
    if last:
        return z[:A.n_rows]
    if h.world is not None:
        lv.plan.exchange(z)
    nxt = h.levels[level + 1]
    rc = nxt.r_lo if lo else nxt.r_hi
    fused_residual_restrict(A, r, z, nxt.f2c, out=rc, tally=tally)
    zc = mg_vcycle(h, level + 1, rc, tally)
    prolong_add(z, zc, nxt.f2c, tally=tally)
    for _ in range(sw.nu2):
        forward_gs_sweep(A, r, z, tally=tally)
    return z[:A.n_rows]
