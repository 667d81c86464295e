"""CPU-side checks of libhpgmxp.so: it loads, exports every declared symbol, and its
host structure functions (the same closed forms the device build kernels run,
csrc/hpg_geom.h) reproduce the reference's setup arrays bitwise."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden
from paper_2507_11512_b200 import _lib
from paper_2507_11512_b200.coloring import greedy_coloring
from paper_2507_11512_b200.comm import HaloPlan  # noqa: F401
from paper_2507_11512_b200.geometry import GlobalProblem, factor_ranks
from paper_2507_11512_b200.problem import host_level

STRUCT = ["s468", "s16", "s8", "odd354", "odd7", "deg144", "deg414", "deg114", "deg111",
          "r2", "r4", "r8", "r8x8", "r3", "r12"]


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "hpgmxp.h")).read()
    declared = set(re.findall(r"\b(hpg_[a-z0-9_]+)\s*\(", hdr))
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    assert L.hpg_abi_version() == 1


def test_factor_ranks():
    assert [factor_ranks(p) for p in (1, 2, 4, 8, 12)] == [(1, 1, 1), (1, 1, 2), (1, 2, 2),
                                                           (2, 2, 2), (2, 2, 3)]


@pytest.mark.parametrize("case", STRUCT)
def test_host_structure_matches_reference(case):
    g = load_golden(f"struct_{case}.npz")
    lx, ly, lz, ranks, levels = map(int, g["dims"])
    gp = GlobalProblem.from_local(lx, ly, lz, ranks)
    for r in range(ranks):
        dom = gp.domain(r)
        for li in range(levels):
            p = f"r{r}_l{li}_"
            vals, cols, nnz, diag, meta = host_level(dom.local_dims, dom.coords, dom.proc_dims)
            np.testing.assert_array_equal(vals, g[p + "values"])
            np.testing.assert_array_equal(cols, g[p + "col_idx"])
            np.testing.assert_array_equal(nnz, g[p + "row_nnz"])
            np.testing.assert_array_equal(diag, g[p + "diag_pos"])
            np.testing.assert_array_equal(meta["color_offsets"], g[p + "color_offsets"])
            assert meta["n_ext"] == int(g[p + "n_ext"])
            assert meta["nnz"] == int(g[p + "row_nnz"].sum())
            col = greedy_coloring(*dom.local_dims)
            np.testing.assert_array_equal(col.perm, g[p + "perm"])
            np.testing.assert_array_equal(col.color, g[p + "color"])
            plan = HaloPlan.__new__(HaloPlan)
            plan.domain = dom
            sends = plan.send_rows()
            assert list(sends) == list(g[p + "neighbors"])
            for nb, rows in sends.items():
                np.testing.assert_array_equal(rows, g[p + f"send_{nb}"])
            if li + 1 < levels:
                dom = dom.coarsen()


@pytest.mark.parametrize("local,ranks,levels", [((8, 8, 8), 8, 4), ((16, 16, 16), 8, 4), ((4, 4, 4), 12, 2),
                                                ((256, 256, 256), 8, 4), ((8, 8, 8), 27, 3)])
def test_peer_memory_staging_layout(local, ranks, levels):
    """Every rank's P2P staging regions (csrc/hpg_p2p.cuh): one per (level, neighbour),
    sized to the neighbour's send list, disjoint, inside the buffer -- checked for the
    8-GPU 2x2x2 grid the driver runs (and 12 / 27 ranks) without GPUs."""
    import ctypes as C
    L = _lib.lib()
    gp = GlobalProblem.from_local(*local, ranks)
    procs = (gp.npx, gp.npy, gp.npz)
    cnt = C.c_int64()
    for R in range(ranks):
        total = L.hpg_host_stage_offset(_lib.ints(*local), _lib.ints(*procs), levels, R, 0, -1, None)
        spans = []
        dom = gp.domain(R)
        for lev in range(levels):
            plan = HaloPlan.__new__(HaloPlan)
            plan.domain = dom
            sends_into_R = {}
            for S in dom.neighbor_ranks():
                sd = gp.domain(S)
                for _ in range(lev):
                    sd = sd.coarsen()
                p2 = HaloPlan.__new__(HaloPlan)
                p2.domain = sd
                sends_into_R[S] = len(p2.send_rows()[R])
            for S in range(ranks):
                off = L.hpg_host_stage_offset(_lib.ints(*local), _lib.ints(*procs), levels, R, lev, S,
                                              C.byref(cnt))
                if S in sends_into_R:
                    assert cnt.value == sends_into_R[S], (R, S, lev)
                    spans.append((off, off + 2 * cnt.value * 8))
                else:
                    assert cnt.value == -1
            if lev + 1 < levels:
                dom = dom.coarsen()
        spans.sort()
        assert spans[0][0] >= 64 * 1024
        for a, b in zip(spans, spans[1:]):
            assert a[1] <= b[0]
        assert spans[-1][1] <= total
