"""CPU oracle for the HPG-MxP solve path.  TEST INFRASTRUCTURE ONLY.

This module is the parity checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it.  The shipped path lives in
``paper_2507_11512_b200`` and fails loudly when its CUDA library is missing.

It restates, in plain numpy, the algorithm of the reference package
``/root/reference/pkg/src/mxpbench`` (abbreviated ``ref:`` below) on the
color-permuted, halo-tailed layout the reference uses, with every
rank of a decomposed problem simulated in lock step inside one process.
Pinning: ``tests/test_oracle.py`` checks this module against the golden
fixtures in ``tests/golden/`` produced by ``tests/golden/make_golden.py``
from the reference itself (bitwise for structure and stencil kernels, the
reference's own frozen iteration counts / residuals for the solver).

Design notes (what is restated, not how the reference spells it):

* Coloring.  The reference's greedy first-fit coloring (ref: coloring.py:49-55)
  on a 27-point lattice reduces to the parity pattern of the local coordinates
  over the axes whose extent is >= 2 (verified against the
  reference in tests).  Rows are ordered by (color, natural index)
  (ref: coloring.py:78-80), so each color block is a sub-lattice in x-fastest
  order and ``iperm`` has a closed form.
* ELL rows keep only in-domain neighbours, ascending global column, padded to
  27 with value 0 / column -1 (ref: problem.py:88-142).  Off-rank columns are
  halo slots laid out neighbour by neighbour in ascending rank id, ascending
  global index (ref: comm.py:180-236).
* Kernels accumulate slot by slot with separate multiply and add
  (ref: krylov.py:76-80, smoother.py:62-75, multigrid.py:107-128); padding
  reads column 0 with value 0 (ref: problem.py:59-65).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

WIDTH = 27
# Stencil offsets in ascending-global-column order: z slowest, x fastest
# (ref: problem.py:22-24).
OFFSETS = [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]

MOTIFS = ("GS", "SpMV", "Ortho", "Restriction", "Prolongation", "Vector ops")


# ----------------------------------------------------------------------------
# geometry (ref: geometry.py:18-180)
# ----------------------------------------------------------------------------

def factor_ranks(p):
    """Most-cubic (a <= b <= c) factorisation of p (ref: geometry.py:18-41)."""
    if p < 1:
        raise ValueError(f"rank count must be >= 1, got {p}")
    triples = [(a, b, p // (a * b))
               for a in range(1, p + 1) if p % a == 0
               for b in range(a, p // a + 1) if (p // a) % b == 0 and p // (a * b) >= b]
    return min(triples, key=lambda t: (t[2] / t[0], t))


@dataclass(frozen=True)
class Box:
    """One rank's box at one level: local dims, rank coords, grid dims."""
    lx: int
    ly: int
    lz: int
    ix: int
    iy: int
    iz: int
    px: int
    py: int
    pz: int

    @property
    def n(self):
        return self.lx * self.ly * self.lz

    @property
    def rank(self):
        return self.ix + self.px * (self.iy + self.py * self.iz)

    @property
    def gdims(self):
        return (self.lx * self.px, self.ly * self.py, self.lz * self.pz)

    @property
    def origin(self):
        return (self.ix * self.lx, self.iy * self.ly, self.iz * self.lz)

    def coarsen(self):
        for name, d in (("x", self.lx), ("y", self.ly), ("z", self.lz)):
            if d % 2:
                raise ValueError(f"axis {name}: local dimension {d} is odd")
        return Box(self.lx // 2, self.ly // 2, self.lz // 2,
                   self.ix, self.iy, self.iz, self.px, self.py, self.pz)

    def neighbours(self):
        """[(rank, (ox, oy, oz))] sorted by rank (ref: geometry.py:159-170)."""
        out = []
        for oz in (-1, 0, 1):
            for oy in (-1, 0, 1):
                for ox in (-1, 0, 1):
                    if ox == oy == oz == 0:
                        continue
                    cx, cy, cz = self.ix + ox, self.iy + oy, self.iz + oz
                    if 0 <= cx < self.px and 0 <= cy < self.py and 0 <= cz < self.pz:
                        out.append((cx + self.px * (cy + self.py * cz), (ox, oy, oz)))
        return sorted(out)


def make_boxes(lx, ly, lz, ranks, dims=None):
    """dims: an explicit (px, py, pz) process grid (default factor_ranks)."""
    px, py, pz = factor_ranks(ranks) if dims is None else dims
    assert px * py * pz == ranks
    return [Box(lx, ly, lz, r % px, (r // px) % py, r // (px * py), px, py, pz)
            for r in range(ranks)]


# ----------------------------------------------------------------------------
# closed-form greedy coloring and permutation (ref: coloring.py:36-123)
# ----------------------------------------------------------------------------

class ColorLayout:
    """Color = parity bits of the active axes; rows sorted by (color, natural)."""

    def __init__(self, lx, ly, lz):
        self.dims = (lx, ly, lz)
        self.active = [a for a in range(3) if self.dims[a] >= 2]
        self.num_colors = 1 << len(self.active) if lx * ly * lz else 0
        sizes = []
        for c in range(self.num_colors):
            par = self.parities(c)
            sizes.append(int(np.prod([(self.dims[a] - par[a] + 1) // 2 for a in range(3)])))
        self.sizes = sizes
        self.offsets = np.zeros(self.num_colors + 1, dtype=np.int64)
        np.cumsum(sizes, out=self.offsets[1:])

    def parities(self, c):
        par = [0, 0, 0]
        for bit, a in enumerate(self.active):
            par[a] = (c >> bit) & 1
        return par

    def color_of(self, x, y, z):
        coords = (x, y, z)
        c = 0
        for bit, a in enumerate(self.active):
            c = c + ((coords[a] & 1) << bit)
        return c

    def iperm(self, x, y, z):
        """natural local coords -> permuted row (vectorised)."""
        x = np.asarray(x, dtype=np.int64)
        y = np.asarray(y, dtype=np.int64)
        z = np.asarray(z, dtype=np.int64)
        c = self.color_of(x, y, z)
        lx, ly, _ = self.dims
        hx = (lx - (x & 1) + 1) // 2
        hy = (ly - (y & 1) + 1) // 2
        return self.offsets[c] + (x >> 1) + hx * ((y >> 1) + hy * (z >> 1))

    def coords(self):
        """(x, y, z) natural local coordinates of every permuted row."""
        lx, ly, lz = self.dims
        n = lx * ly * lz
        nat = np.arange(n, dtype=np.int64)
        x, y, z = nat % lx, (nat // lx) % ly, nat // (lx * ly)
        p = self.iperm(x, y, z)
        out = np.empty((3, n), dtype=np.int64)
        out[0, p], out[1, p], out[2, p] = x, y, z
        return out


# ----------------------------------------------------------------------------
# one rank-level: ELL operand + halo plan (ref: problem.py:88-175, comm.py:180-236)
# ----------------------------------------------------------------------------

def _region(box, o, outside):
    """Box-shaped region next to face/edge/corner ``o``: outside (halo) or inside (send)."""
    rng = []
    for d, off in zip((box.lx, box.ly, box.lz), o):
        if off == 0:
            rng.append(np.arange(d))
        elif off > 0:
            rng.append(np.array([d if outside else d - 1]))
        else:
            rng.append(np.array([-1 if outside else 0]))
    z, y, x = np.meshgrid(rng[2], rng[1], rng[0], indexing="ij")
    return x.ravel(), y.ravel(), z.ravel()


@dataclass
class RankLevel:
    box: Box
    layout: ColorLayout
    values: np.ndarray          # [n, 27] float64 (compacted, padded)
    col_idx: np.ndarray         # [n, 27] int32, padding -1, halo >= n
    row_nnz: np.ndarray
    diag_pos: np.ndarray
    neighbours: list            # [(rank, offset)]
    send_rows: dict             # rank -> permuted rows, peer request order
    recv_slices: dict           # rank -> slice into the halo tail
    halo_size: int
    f2c: np.ndarray = None      # coarse row -> parent (finer) row
    _lo: np.ndarray = field(default=None, repr=False)

    @property
    def n(self):
        return self.box.n

    @property
    def n_ext(self):
        return self.box.n + self.halo_size

    @property
    def nnz(self):
        return int(self.row_nnz.sum())

    @property
    def values_lo(self):
        if self._lo is None:
            self._lo = self.values.astype(np.float32)
        return self._lo

    def vals(self, dtype):
        return self.values_lo if np.dtype(dtype) == np.float32 else self.values

    def safe_cols(self):
        cache = self.__dict__.setdefault("_safe", None)
        if cache is None:
            cache = np.where(self.col_idx >= 0, self.col_idx, 0)
            self.__dict__["_safe"] = cache
        return cache

    def sweep_operands(self, dtype):
        """(off-diagonal values, diagonal, safe columns), cached per dtype."""
        key = np.dtype(dtype).str
        cache = self.__dict__.setdefault("_sweep", {})
        if key not in cache:
            A = self.vals(dtype)
            rows = np.arange(self.n)
            off = A.copy()
            off[rows, self.diag_pos] = 0
            diag = A[rows, self.diag_pos].copy()
            if np.any(diag == 0):
                raise ZeroDivisionError("zero diagonal entry in smoother input")
            cache[key] = (off, diag, self.safe_cols())
        return cache[key]

    def row_has_halo(self):
        return (self.col_idx >= self.n).any(axis=1)


def build_rank_level(box):
    lay = ColorLayout(box.lx, box.ly, box.lz)
    n = box.n
    gx, gy, gz = box.gdims
    ox, oy, oz = box.origin
    x, y, z = lay.coords()
    nbrs = box.neighbours()

    # halo slot base per neighbour, ascending rank id (ref: comm.py:219-227)
    base = {}
    nxt = n
    regions = {}
    for rk, o in nbrs:
        rx, ry, rz = _region(box, o, outside=True)
        regions[o] = (rx, ry, rz)
        base[o] = nxt
        nxt += len(rx)
    halo_size = nxt - n

    vals = np.zeros((n, WIDTH))
    cols = np.full((n, WIDTH), -1, dtype=np.int64)
    valid = np.zeros((n, WIDTH), dtype=bool)
    for s, (dx, dy, dz) in enumerate(OFFSETS):
        ax, ay, az = x + dx, y + dy, z + dz
        ok = ((0 <= ax + ox) & (ax + ox < gx) & (0 <= ay + oy) & (ay + oy < gy)
              & (0 <= az + oz) & (az + oz < gz))
        inside = ((0 <= ax) & (ax < box.lx) & (0 <= ay) & (ay < box.ly)
                  & (0 <= az) & (az < box.lz))
        col = np.full(n, -1, dtype=np.int64)
        own = ok & inside
        col[own] = lay.iperm(ax[own], ay[own], az[own])
        off = ok & ~inside
        if off.any():
            # which neighbour face/edge/corner, and position within its region
            sx = np.where(ax < 0, -1, np.where(ax >= box.lx, 1, 0))
            sy = np.where(ay < 0, -1, np.where(ay >= box.ly, 1, 0))
            sz = np.where(az < 0, -1, np.where(az >= box.lz, 1, 0))
            for o in base:
                m = off & (sx == o[0]) & (sy == o[1]) & (sz == o[2])
                if not m.any():
                    continue
                wx = box.lx if o[0] == 0 else 1
                wy = box.ly if o[1] == 0 else 1
                px_ = np.where(o[0] == 0, ax[m], 0)
                py_ = np.where(o[1] == 0, ay[m], 0)
                pz_ = np.where(o[2] == 0, az[m], 0)
                col[m] = base[o] + px_ + wx * (py_ + wy * pz_)
        valid[:, s] = ok
        cols[:, s] = col
        vals[:, s] = np.where(ok, 26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0, 0.0)

    # compact: valid entries first, order preserved (ref: problem.py:127-138)
    order = np.argsort(~valid, axis=1, kind="stable")
    vals = np.take_along_axis(vals, order, axis=1)
    cols = np.take_along_axis(cols, order, axis=1)
    row_nnz = valid.sum(axis=1)
    pad = np.arange(WIDTH)[None, :] >= row_nnz[:, None]
    vals[pad] = 0.0
    cols[pad] = -1
    diag_pos = valid[:, :13].sum(axis=1)

    send_rows, recv_slices = {}, {}
    for rk, o in nbrs:
        sx_, sy_, sz_ = _region(box, o, outside=False)
        send_rows[rk] = lay.iperm(sx_, sy_, sz_).astype(np.int64)
        cnt = len(regions[o][0])
        recv_slices[rk] = slice(base[o], base[o] + cnt)
    return RankLevel(box=box, layout=lay, values=vals, col_idx=cols.astype(np.int32),
                     row_nnz=row_nnz.astype(np.int32), diag_pos=diag_pos.astype(np.int32),
                     neighbours=nbrs, send_rows=send_rows, recv_slices=recv_slices,
                     halo_size=halo_size)


def injection_map(coarse, fine):
    """coarse permuted row -> fine permuted row of point (2x,2y,2z) (ref: multigrid.py:87-99)."""
    cx, cy, cz = coarse.layout.coords()
    return fine.layout.iperm(2 * cx, 2 * cy, 2 * cz).astype(np.int64)


# ----------------------------------------------------------------------------
# distributed world simulated in lock step
# ----------------------------------------------------------------------------

class World:
    """All ranks of one problem; vectors are lists of per-rank arrays."""

    def __init__(self, lx, ly, lz, ranks, levels, dims=None):
        self.ranks = ranks
        boxes = make_boxes(lx, ly, lz, ranks, dims)
        self.levels = []           # levels[l][rank] -> RankLevel
        for lev in range(levels):
            per = [build_rank_level(b) for b in boxes]
            if lev > 0:
                for r in range(ranks):
                    per[r].f2c = injection_map(per[r], self.levels[-1][r])
            self.levels.append(per)
            if lev + 1 < levels:
                boxes = [b.coarsen() for b in boxes]

    # -- comm (ref: comm.py:239-279) --------------------------------------
    def exchange(self, lev, vs):
        L = self.levels[lev]
        if self.ranks == 1:
            return
        sends = {}
        for r in range(self.ranks):
            for nb in L[r].send_rows:
                sends[(r, nb)] = vs[r][L[r].send_rows[nb]].copy()
        for r in range(self.ranks):
            for nb, sl in L[r].recv_slices.items():
                vs[r][sl] = sends[(nb, r)]

    def allreduce(self, parts):
        """Ascending-rank fold, identical on every rank (ref: comm.py:97-108)."""
        acc = parts[0].copy() if isinstance(parts[0], np.ndarray) else parts[0]
        for p in parts[1:]:
            acc = acc + p
        return acc


# ----------------------------------------------------------------------------
# stencil kernels (ref: krylov.py:76-107, smoother.py:62-114, multigrid.py:102-137)
# ----------------------------------------------------------------------------

_POOL = None
_THREADS = 1


def set_threads(k):
    """Split the row loops over k host threads (numpy releases the GIL in the
    gathers and ufuncs).  Per-row arithmetic is unchanged, so results are
    bitwise identical for any k; used for the CPU baseline timing."""
    global _POOL, _THREADS
    from concurrent.futures import ThreadPoolExecutor
    _THREADS = max(1, int(k))
    _POOL = ThreadPoolExecutor(_THREADS) if _THREADS > 1 else None


def _rows_parallel(fn, nrows):
    """fn(a, b) over row chunks; results concatenated in row order."""
    if _POOL is None or nrows < 4096 * _THREADS:
        return fn(0, nrows)
    cuts = [nrows * t // _THREADS for t in range(_THREADS + 1)]
    parts = list(_POOL.map(lambda t: fn(cuts[t], cuts[t + 1]), range(_THREADS)))
    return np.concatenate(parts)


def row_products(vals, cols, x):
    """sum_s vals[:, s] * x[cols[:, s]], slot by slot, separate mul and add."""
    def part(a, b):
        acc = np.zeros(b - a, dtype=x.dtype)
        v, c = vals[a:b], cols[a:b]
        for s in range(vals.shape[1]):
            acc += v[:, s] * x[c[:, s]]
        return acc
    return _rows_parallel(part, vals.shape[0])


def spmv_rank(lv, x):
    return row_products(lv.vals(x.dtype), lv.safe_cols(), x)


def gs_sweep_rank(lv, r, z):
    """Forward multicolor GS over z (halo-tailed), in place (ref: smoother.py:78-112)."""
    off, diag, cols = lv.sweep_operands(z.dtype)
    offs = lv.layout.offsets
    for c in range(lv.layout.num_colors):
        a, b = int(offs[c]), int(offs[c + 1])
        acc = row_products(off[a:b], cols[a:b], z)
        z[a:b] = (r[a:b] - acc) / diag[a:b]


def restrict_rank(lv_f, lv_c, r_f, z_f):
    """r_c = (r_f - A_f z_f)[f2c] evaluated only at injected rows (ref: multigrid.py:107-128)."""
    rows = lv_c.f2c
    A = lv_f.vals(z_f.dtype)[rows]
    acc = row_products(A, lv_f.safe_cols()[rows], z_f)
    return r_f[rows] - acc


def prolong_rank(lv_c, z_f, z_c):
    z_f[lv_c.f2c] += z_c


# ----------------------------------------------------------------------------
# metrics (ref: metrics.py:37-108)
# ----------------------------------------------------------------------------

def kernel_flops(kernel, **s):
    return {
        "spmv": lambda: 2 * s.get("nnz", 0),
        "gs_sweep": lambda: 2 * s.get("nnz", 0),
        "dot": lambda: 2 * s.get("n", 0),
        "norm": lambda: 2 * s.get("n", 0),
        "scale": lambda: s.get("n", 0),
        "vsub": lambda: s.get("n", 0),
        "vadd": lambda: s.get("n", 0),
        "waxpby": lambda: 3 * s.get("n", 0),
        "cgs2": lambda: 8 * s.get("n", 0) * s.get("k", 0) + 2 * s.get("n", 0),
        "gemv_update": lambda: 2 * s.get("n", 0) * s.get("k", 0),
        "restrict_fused": lambda: 2 * s.get("nnz", 0) + s.get("n_c", 0),
        "restrict_inject": lambda: 0,
        "prolong_add": lambda: s.get("n_c", 0),
    }[kernel]()


def kernel_bytes(kernel, w, **s):
    n, k, nnz, nc = s.get("n", 0), s.get("k", 0), s.get("nnz", 0), s.get("n_c", 0)
    return {
        "spmv": nnz * (w + 4) + 2 * n * w,
        "gs_sweep": nnz * (w + 4) + 3 * n * w,
        "dot": 2 * n * w,
        "norm": n * w,
        "scale": 2 * n * w,
        "vsub": 3 * n * w,
        "vadd": 3 * n * w,
        "waxpby": 3 * n * w,
        "cgs2": 4 * n * k * w + 4 * n * w,
        "gemv_update": (n * k + 2 * n) * w,
        "restrict_fused": nnz * (2 * w + 4) + 2 * nc * w,
        "restrict_inject": 2 * nc * w,
        "prolong_add": 3 * nc * w,
    }[kernel]


KERNEL_MOTIF = {"spmv": "SpMV", "gs_sweep": "GS", "dot": "Vector ops", "norm": "Vector ops",
                "scale": "Vector ops", "vsub": "Vector ops", "vadd": "Vector ops",
                "waxpby": "Vector ops", "cgs2": "Ortho", "gemv_update": "Ortho",
                "restrict_fused": "Restriction", "restrict_inject": "Restriction",
                "prolong_add": "Prolongation"}


class Count:
    """Per-motif flop/byte accumulator for ONE rank (ref: metrics.py:111-143)."""

    def __init__(self):
        self.flops = {m: 0 for m in MOTIFS}
        self.bytes = {m: 0 for m in MOTIFS}

    def add(self, kernel, dtype, motif=None, **s):
        m = motif or KERNEL_MOTIF[kernel]
        self.flops[m] += int(kernel_flops(kernel, **s))
        self.bytes[m] += int(kernel_bytes(kernel, np.dtype(dtype).itemsize, **s))


def penalty_factor(n_d, n_ir):
    if n_d < 1 or n_ir < 1:
        raise ValueError(f"iteration counts must be >= 1, got ({n_d}, {n_ir})")
    return min(1.0, n_d / n_ir)


# ----------------------------------------------------------------------------
# V-cycle (ref: multigrid.py:140-171) over all ranks
# ----------------------------------------------------------------------------

class Solver:
    def __init__(self, lx, ly, lz, ranks=1, levels=4, nu1=1, nu2=1, nu_c=1, dims=None):
        self.world = World(lx, ly, lz, ranks, levels, dims)
        self.nlev = levels
        self.nu1, self.nu2, self.nu_c = nu1, nu2, nu_c
        self.count = Count()        # rank 0's tally (counts are per rank)

    @property
    def ranks(self):
        return self.world.ranks

    def L(self, lev):
        return self.world.levels[lev]

    def gs_sweep(self, lev, r, z, z_is_zero):
        L = self.L(lev)
        if z_is_zero:
            for zz in z:
                zz[:] = 0
        else:
            self.world.exchange(lev, z)
        for q in range(self.ranks):
            gs_sweep_rank(L[q], r[q], z[q])
        self.count.add("gs_sweep", z[0].dtype, nnz=L[0].nnz, n=L[0].n)

    def vcycle(self, r, lev=0):
        """r: list of per-rank owned vectors; returns list of owned z (copies)."""
        L = self.L(lev)
        dt = r[0].dtype
        z = [np.zeros(lv.n_ext, dtype=dt) for lv in L]
        last = lev == self.nlev - 1
        for s in range(self.nu_c if last else self.nu1):
            self.gs_sweep(lev, r, z, z_is_zero=(s == 0))
        if last:
            return [zz[:lv.n].copy() for zz, lv in zip(z, L)]
        self.world.exchange(lev, z)
        C = self.L(lev + 1)
        rc = [restrict_rank(L[q], C[q], r[q], z[q]) for q in range(self.ranks)]
        self.count.add("restrict_fused", dt, nnz=int(L[0].row_nnz[C[0].f2c].sum()), n_c=C[0].n)
        zc = self.vcycle(rc, lev + 1)
        for q in range(self.ranks):
            prolong_rank(C[q], z[q], zc[q])
        self.count.add("prolong_add", dt, n_c=C[0].n)
        for _ in range(self.nu2):
            self.gs_sweep(lev, r, z, z_is_zero=False)
        return [zz[:lv.n].copy() for zz, lv in zip(z, L)]

    def spmv(self, x_ext, lev=0):
        self.world.exchange(lev, x_ext)
        L = self.L(lev)
        out = [spmv_rank(L[q], x_ext[q]) for q in range(self.ranks)]
        self.count.add("spmv", x_ext[0].dtype, nnz=L[0].nnz, n=L[0].n)
        return out

    def rhs(self):
        """b = A 1 = row sums, per rank (ref: problem.py:152-162)."""
        return [lv.values.sum(axis=1) for lv in self.L(0)]

    # -- GMRES / GMRES-IR (ref: krylov.py:110-308) -------------------------
    def gmres(self, b, mode="double", tol=1e-9, max_iters=300, m=30, x0=None,
              precond=True):
        if mode not in ("double", "mixed"):
            raise ValueError(f"unknown mode: {mode!r}")
        dt = np.float32 if mode == "mixed" else np.float64
        R = self.ranks
        L0 = self.L(0)
        n = [lv.n for lv in L0]
        N = n[0]
        x = [np.zeros(lv.n_ext) for lv in L0]
        if x0 is not None:
            for q in range(R):
                x[q][:n[q]] = x0[q]
        zt = [np.zeros(lv.n_ext, dtype=dt) for lv in L0]
        Q = [np.zeros((m + 1, n[q]), dtype=dt) for q in range(R)]
        H = np.zeros((m + 1, m), dtype=dt)
        t = np.zeros(m + 1, dtype=dt)
        cs = np.zeros(m + 1, dtype=dt)
        sn = np.zeros(m + 1, dtype=dt)
        M = (lambda v: self.vcycle(v)) if precond else (lambda v: [a.copy() for a in v])

        def true_residual():
            y = self.spmv(x)
            r = [b[q] - y[q] for q in range(R)]
            rho = float(np.sqrt(self.world.allreduce([rr @ rr for rr in r])))
            self.count.add("vsub", np.float64, n=N)
            self.count.add("norm", np.float64, n=N)
            return r, rho

        rho0 = float(np.sqrt(self.world.allreduce([bb @ bb for bb in b])))
        self.count.add("norm", np.float64, n=N)
        res = {"iterations": 0, "restarts": 0, "relres": 0.0, "converged": True,
               "cycle_iters": [], "pairs": []}
        if rho0 == 0.0:
            return res, [xx[:nn].copy() for xx, nn in zip(x, n)]
        total = cycles = 0
        last_rec = None
        converged = False
        relres = 1.0
        while True:
            r, rho = true_residual()
            relres = rho / rho0
            if cycles > 0 and last_rec is not None:
                res["pairs"].append((last_rec, rho))
            if relres < tol:
                converged = True
                break
            if total >= max_iters:
                break
            for q in range(R):
                Q[q][0] = r[q] / rho
            self.count.add("scale", np.float64, n=N)
            t[:] = 0
            t[0] = rho
            H[:] = 0
            cs[:] = 0
            sn[:] = 0
            rho_rec = rho
            k = 0
            broke = False
            while k < m and total < max_iters and rho_rec / rho0 >= tol:
                zv = M([Q[q][k] for q in range(R)])
                for q in range(R):
                    zt[q][:n[q]] = zv[q]
                w = self.spmv(zt)
                kb = k + 1
                for _ in range(2):       # CGS2 (ref: krylov.py:110-129)
                    h = self.world.allreduce([Q[q][:kb] @ w[q] for q in range(R)])
                    for q in range(R):
                        w[q] -= Q[q][:kb].T @ h
                    H[:kb, k] += h
                self.count.add("cgs2", dt, n=N, k=kb)
                beta = np.sqrt(self.world.allreduce([ww @ ww for ww in w]))
                H[k + 1, k] = beta
                for q in range(R):
                    Q[q][k + 1] = w[q] / beta if beta != 0 else 0
                self.count.add("norm", dt, motif="Ortho", n=N)
                self.count.add("scale", dt, motif="Ortho", n=N)
                try:
                    rho_rec = givens_update(H, t, cs, sn, k)
                except ZeroDivisionError:
                    broke = True
                    break
                k += 1
                total += 1
            if k > 0:
                y = back_substitute(H, t, k)
                ru = [Q[q][:k].T @ y.astype(dt) for q in range(R)]
                self.count.add("gemv_update", dt, n=N, k=k)
                zu = M(ru)
                for q in range(R):
                    x[q][:n[q]] += zu[q]
                self.count.add("vadd", np.float64, n=N)
            res["cycle_iters"].append(k)
            cycles += 1
            last_rec = rho_rec
            if broke:
                _, rho = true_residual()
                relres = rho / rho0
                converged = relres < tol
                break
        res.update(iterations=total, restarts=cycles, relres=relres, converged=converged)
        return res, [xx[:nn].copy() for xx, nn in zip(x, n)]


def givens_update(H, t, c, s, k):
    """fp64 rotation on promoted values, stored at the arrays' dtype (ref: krylov.py:132-159)."""
    col = H[:k + 2, k].astype(np.float64)
    for j in range(k):
        a, b_ = col[j], col[j + 1]
        cj, sj = float(c[j]), float(s[j])
        col[j] = cj * a + sj * b_
        col[j + 1] = -sj * a + cj * b_
    mu = float(np.hypot(col[k], col[k + 1]))
    if mu == 0.0:
        raise ZeroDivisionError(f"zero pivot at column {k}")
    ck, sk = col[k] / mu, col[k + 1] / mu
    col[k], col[k + 1] = mu, 0.0
    H[:k + 2, k] = col
    c[k], s[k] = ck, sk
    tk = float(t[k])
    t[k] = ck * tk
    t[k + 1] = -sk * tk
    return abs(float(t[k + 1]))


def back_substitute(H, t, k):
    """k x k upper-triangular solve on fp64 promotions (ref: krylov.py:162-169)."""
    R = H[:k, :k].astype(np.float64)
    rhs = t[:k].astype(np.float64)
    y = np.zeros(k)
    for i in reversed(range(k)):
        y[i] = (rhs[i] - R[i, i + 1:k] @ y[i + 1:k]) / R[i, i]
    return y


# ----------------------------------------------------------------------------
# validation + penalty (ref: bench.py:139-183, metrics.py:98-102)
# ----------------------------------------------------------------------------

def run_validation(lx, ly, lz, ranks=1, levels=4, tol=1e-9, nd_cap=10000, m=30,
                   mode="standard", dims=None):
    s = Solver(lx, ly, lz, ranks, levels, dims=dims)
    b = s.rhs()
    dres, _ = s.gmres(b, "double", tol, nd_cap, m)
    if mode == "standard":
        if not dres["converged"]:
            raise RuntimeError("double GMRES did not converge")
        target = tol
    else:
        target = dres["relres"] if not dres["converged"] else tol
    mres, _ = s.gmres(b, "mixed", target, nd_cap, m)
    return {"mode": mode, "n_d": dres["iterations"], "n_ir": mres["iterations"],
            "ratio": dres["iterations"] / mres["iterations"], "residual": dres["relres"]}
