"""Pin the CPU oracle (oracle/hpgmxp_oracle.py) against the reference's fixtures.

The fixtures in tests/golden/ were produced by importing the reference package
(tests/golden/make_golden.py).  Structure and stencil kernels must match
bitwise; solver iteration counts follow the reference's own frozen values
(ref tests: test_krylov.py:221-232, test_acceptance.py:158-160, 347-348,
test_bench.py:70-86) and the envelope recorded in tests/golden/solves.json.
"""

import numpy as np
import pytest

import hpgmxp_oracle as O
from conftest import load_golden

STRUCT = ["s468", "s16", "s8", "odd354", "odd7", "deg144", "deg414", "deg114", "deg111",
          "r2", "r4", "r8", "r8x8", "r3", "r12",
          # explicit process grids that split x (tests/golden/make_golden.py XSPLIT_STRUCT)
          "x211", "x221", "x212", "x411"]


def _dims(g):
    return tuple(int(d) for d in g["proc_dims"]) if "proc_dims" in g else None


def test_factor_ranks_matches_reference_table():
    # ref: tests/test_geometry.py:11-17 and SURVEY.md 2
    assert O.factor_ranks(1) == (1, 1, 1)
    assert O.factor_ranks(2) == (1, 1, 2)
    assert O.factor_ranks(4) == (1, 2, 2)
    assert O.factor_ranks(8) == (2, 2, 2)
    assert O.factor_ranks(12) == (2, 2, 3)
    assert O.factor_ranks(7) == (1, 1, 7)


@pytest.mark.parametrize("case", STRUCT)
def test_structure_bitwise(case):
    g = load_golden(f"struct_{case}.npz")
    lx, ly, lz, ranks, levels = map(int, g["dims"])
    w = O.World(lx, ly, lz, ranks, levels, _dims(g))
    for r in range(ranks):
        for li in range(levels):
            p = f"r{r}_l{li}_"
            lv = w.levels[li][r]
            np.testing.assert_array_equal(lv.values, g[p + "values"])
            np.testing.assert_array_equal(lv.col_idx, g[p + "col_idx"])
            np.testing.assert_array_equal(lv.row_nnz, g[p + "row_nnz"])
            np.testing.assert_array_equal(lv.diag_pos, g[p + "diag_pos"])
            np.testing.assert_array_equal(lv.layout.offsets, g[p + "color_offsets"])
            assert lv.n_ext == int(g[p + "n_ext"])
            if li > 0:
                np.testing.assert_array_equal(lv.f2c, g[p + "f2c"])
            nbs = [rk for rk, _ in lv.neighbours]
            np.testing.assert_array_equal(np.array(nbs, dtype=np.int64), g[p + "neighbors"])
            for nb in nbs:
                np.testing.assert_array_equal(lv.send_rows[nb], g[p + f"send_{nb}"])
                sl = lv.recv_slices[nb]
                assert [sl.start, sl.stop] == list(g[p + f"recv_{nb}"])


@pytest.mark.parametrize("case", ["k16", "k8r8", "k8x8r8", "k8r2", "kx211", "kx221", "kx212"])
def test_kernels_bitwise(case):
    g = load_golden(f"kernels_{case}.npz")
    l, _, _, ranks, levels = map(int, g["dims"])
    s = O.Solver(l, l, l, ranks, levels, dims=_dims(g))
    L0, L1 = s.L(0), s.L(1)
    for tag, dt in (("f64", np.float64), ("f32", np.float32)):
        xs = [g[f"r{q}_{tag}_x"] for q in range(ranks)]
        rs = [g[f"r{q}_{tag}_r"] for q in range(ranks)]

        def ext(v, q):
            out = np.zeros(L0[q].n_ext, dtype=dt)
            out[:L0[q].n] = v
            return out

        y = s.spmv([ext(xs[q], q) for q in range(ranks)])
        z0 = [np.zeros(L0[q].n_ext, dtype=dt) for q in range(ranks)]
        s.gs_sweep(0, rs, z0, z_is_zero=True)
        z1 = [ext(xs[q], q) for q in range(ranks)]
        s.gs_sweep(0, rs, z1, z_is_zero=False)
        x3 = [ext(xs[q], q) for q in range(ranks)]
        s.world.exchange(0, x3)
        vc = s.vcycle([r.copy() for r in rs])
        for q in range(ranks):
            assert y[q].dtype == dt
            np.testing.assert_array_equal(y[q], g[f"r{q}_{tag}_spmv"])
            np.testing.assert_array_equal(z0[q][:L0[q].n], g[f"r{q}_{tag}_gs0"])
            np.testing.assert_array_equal(z1[q][:L0[q].n], g[f"r{q}_{tag}_gs1"])
            rc = O.restrict_rank(L0[q], L1[q], rs[q], x3[q])
            np.testing.assert_array_equal(rc, g[f"r{q}_{tag}_restrict"])
            xf = ext(xs[q], q)
            O.prolong_rank(L1[q], xf, g[f"r{q}_{tag}_xc"])
            np.testing.assert_array_equal(xf[:L0[q].n], g[f"r{q}_{tag}_prolong"])
            np.testing.assert_array_equal(vc[q], g[f"r{q}_{tag}_vcycle"])


def test_flop_and_byte_model_matches_reference_formulas():
    # ref: metrics.py:37-77 ; SURVEY.md 8(d) per-cycle numbers at 256^3
    n = 256 ** 3
    nnz = (3 * 256 - 2) ** 3
    assert O.kernel_flops("spmv", nnz=nnz, n=n) == 2 * nnz
    assert O.kernel_bytes("gs_sweep", 4, nnz=nnz, n=n) == nnz * 8 + 3 * n * 4
    assert O.kernel_bytes("cgs2", 8, n=n, k=3) == 4 * n * 3 * 8 + 4 * n * 8
    assert O.kernel_flops("cgs2", n=n, k=3) == 8 * n * 3 + 2 * n
    assert O.penalty_factor(2305, 2382) == pytest.approx(0.968, abs=1e-3)
    assert O.penalty_factor(30, 20) == 1.0


def _solves():
    return load_golden("solves.json")


def test_solve_16_double_frozen_counts():
    # ref: tests/test_krylov.py:221-225 -> 16 iterations, relres 4.4911594142630304e-10
    s = O.Solver(16, 16, 16, 1, 4)
    res, x = s.gmres(s.rhs(), "double")
    assert res["converged"] and res["iterations"] == 16
    assert res["relres"] == pytest.approx(4.4911594142630304e-10, rel=1e-6)
    gx = load_golden("solves_x.npz")["l16_1_double"]
    np.testing.assert_allclose(x[0], gx, rtol=0, atol=1e-12)


def test_solve_16_mixed_frozen_counts():
    # ref: tests/test_krylov.py:228-232 -> 20 iterations; envelope from solves.json
    s = O.Solver(16, 16, 16, 1, 4)
    res, x = s.gmres(s.rhs(), "mixed")
    env = [_solves()["l16"][t]["mixed"]["iterations"] for t in ("1", "default")]
    assert res["converged"] and res["relres"] <= 1e-9
    assert min(env) - 1 <= res["iterations"] <= max(env) + 1
    assert res["cycle_iters"][0] == _solves()["l16"]["1"]["mixed"]["cycle_iters"][0]


def test_restarted_small_solve():
    # ref: tests/test_krylov.py:145-155: unpreconditioned 4^3, random rhs (seed 42,
    # natural order), m=5, tol 1e-10 -> 4 restarts, 18 iterations.  The oracle
    # works in the color-permuted order, so permute the rhs the same way.
    s = O.Solver(4, 4, 4, 1, 1)
    x, y, z = s.L(0)[0].layout.coords()
    b_nat = np.random.default_rng(42).standard_normal(64)
    res, _ = s.gmres([b_nat[x + 4 * (y + 4 * z)]], "double", tol=1e-10, m=5, precond=False)
    assert res["converged"] and res["restarts"] == 4 and res["iterations"] == 18


def test_fullscale_validation_tiny():
    # ref: tests/test_bench.py:80-86 -> 8^3 fullscale, 1 rank: 10 / 13, 3.338933745599345e-11
    v = O.run_validation(8, 8, 8, 1, 4, mode="fullscale")
    assert v["n_d"] == 10 and v["n_ir"] == 13
    assert v["residual"] == pytest.approx(3.338933745599345e-11, rel=1e-6)


@pytest.mark.slow
def test_solve_8_ranks_counts():
    # ref: tests/test_acceptance.py:347-348 -> 8 ranks x 8^3: 18 double / 23 mixed
    s = O.Solver(8, 8, 8, 8, 4)
    b = s.rhs()
    d, _ = s.gmres(b, "double")
    mx, _ = s.gmres(b, "mixed")
    assert d["iterations"] == 18
    env = [_solves()["r8l8"][t]["mixed"]["iterations"] for t in ("1", "default")]
    assert min(env) - 1 <= mx["iterations"] <= max(env) + 1


def test_validation_standard_small():
    # ref: tests/test_bench.py:70-77 -> 4^3 (3 levels): n_d 6, n_ir 8, residual 8.99325262264748e-12
    v = O.run_validation(4, 4, 4, 1, 3)
    assert v["n_d"] == 6 and v["n_ir"] in (7, 8, 9)
    assert v["residual"] == pytest.approx(8.99325262264748e-12, rel=1e-6)


def test_threaded_oracle_is_bitwise_identical():
    """The CPU-baseline timing splits row loops over threads: same bits."""
    s = O.Solver(16, 16, 16, 1, 4)
    r = np.random.default_rng(3).standard_normal(4096)
    a = s.vcycle([r.copy()])[0]
    O.set_threads(4)
    try:
        b = s.vcycle([r.copy()])[0]
    finally:
        O.set_threads(1)
    np.testing.assert_array_equal(a, b)


@pytest.mark.slow
@pytest.mark.parametrize("case", ["x211l16", "x221l8", "x212l8"])
def test_xsplit_solve_counts(case):
    """x-splitting process grids: fp64 counts exact, mixed per cycle within the
    reference envelope +-1 (tests/golden/solves_xsplit.json, from the reference)."""
    gold = load_golden("solves_xsplit.json")[case]
    l = int(case[5:])
    dims = tuple(int(c) for c in case[1:4])
    ranks = dims[0] * dims[1] * dims[2]
    s = O.Solver(l, l, l, ranks, 4, dims=dims)
    b = s.rhs()
    d, _ = s.gmres(b, "double")
    assert d["iterations"] == gold["1"]["double"]["iterations"]
    mx, _ = s.gmres(b, "mixed")
    refs = [gold[t]["mixed"]["cycle_iters"] for t in ("1", "default")]
    assert all(len(r) == len(mx["cycle_iters"]) for r in refs)
    for i, g in enumerate(mx["cycle_iters"]):
        assert min(r[i] for r in refs) - 1 <= g <= max(r[i] for r in refs) + 1


def test_reduction_envelope_pinned_to_reference():
    """tests/golden/reduction_envelope.json (make_envelope.py): its OpenBLAS-GEMV
    order -- the reference's own expressions run by the oracle -- reproduces the
    reference's recorded per-cycle counts, and every order agrees on cycle 1."""
    env = load_golden("reduction_envelope.json")
    gold = dict(load_golden("solves.json"), **load_golden("solves_xsplit.json"))
    for case, orders in env.items():
        runs = [gold[case][t]["mixed"]["cycle_iters"] for t in ("1", "default")]
        assert orders["blas_gemv"] in runs, (case, orders["blas_gemv"], runs)
        assert len({tuple(o[:1]) for o in orders.values()}) == 1, (case, orders)
