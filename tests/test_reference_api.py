"""The reference's array API, called the way the reference's own tests call it
(host numpy vectors in and out, in-place mutation), against the device
implementation.  Each test restates one case of /root/reference/pkg/tests
(file:line cited); the device does the arithmetic, host arrays are copied in
and written back like the reference's in-place contracts.

Deviations, by design: operands live on the device (``generate_matrix`` returns
a device level whose off-rank columns already hold halo slots); ranks are
processes (the RankWorld thread cases are covered by tests/test_multigpu.py).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _seq_spmv(values, col_idx, x):
    """Row-by-row, slot-ordered y = A x, padding -> column 0 (restated from
    ref tests/_oracles.py seq_spmv)."""
    y = np.zeros(values.shape[0], dtype=x.dtype)
    for i in range(values.shape[0]):
        acc = x.dtype.type(0)
        for s in range(values.shape[1]):
            c = col_idx[i, s]
            acc = acc + values[i, s] * x[c if c >= 0 else 0]
        y[i] = acc
    return y


def _seq_gs(values, col_idx, diag_pos, r, z):
    """Sequential forward Gauss-Seidel in row order (ref tests/_oracles.py seq_gs_sweep)."""
    for i in range(values.shape[0]):
        acc = z.dtype.type(0)
        for s in range(values.shape[1]):
            c = col_idx[i, s]
            v = z.dtype.type(0) if s == diag_pos[i] else values[i, s]
            acc = acc + v * z[c if c >= 0 else 0]
        z[i] = (r[i] - acc) / values[i, diag_pos[i]]


def _single_rank_system(nx, ny, nz):
    from paper_2507_11512_b200.geometry import GlobalProblem
    from paper_2507_11512_b200.problem import generate_matrix, generate_rhs
    A = generate_matrix(GlobalProblem.from_local(nx, ny, nz, 1).domain(0))
    return A, generate_rhs(A)


def _permuted(nx, ny, nz):
    from paper_2507_11512_b200.coloring import color, permute_system
    from paper_2507_11512_b200.comm import build_halo_plan
    from paper_2507_11512_b200.geometry import GlobalProblem
    from paper_2507_11512_b200.problem import generate_matrix
    dom = GlobalProblem.from_local(nx, ny, nz, 1).domain(0)
    A = generate_matrix(dom)
    c = color(A, "greedy")
    Ap, _ = permute_system(A, [], c)
    build_halo_plan(dom, Ap)
    return Ap, c


def _hierarchy(l, levels, sweeps=None):
    from paper_2507_11512_b200.geometry import GlobalProblem
    from paper_2507_11512_b200.multigrid import build_hierarchy
    from paper_2507_11512_b200.smoother import SmootherWorkspace
    return build_hierarchy(GlobalProblem.from_local(l, l, l, 1).domain(0), levels,
                           sweeps=sweeps or SmootherWorkspace())


# ---------------------------------------------------------------- problem / coloring

def test_generate_matrix_row_classes_and_order():
    # ref: tests/test_problem.py:18-57 (nnz classes 8/12/18/27, diagonal 26 at diag_pos,
    # entries ascending in global column)
    A, vecs = _single_rank_system(4, 4, 4)
    counts = dict(zip(*np.unique(A.row_nnz, return_counts=True)))
    assert counts == {8: 8, 12: 24, 18: 24, 27: 8}
    assert np.all(A.values[np.arange(64), A.diag_pos] == 26.0)
    g = A.col_global
    for i in range(A.n_rows):
        row = g[i, :A.row_nnz[i]]
        assert np.all(np.diff(row) > 0) and np.all(g[i, A.row_nnz[i]:] == -1)
    b = vecs.b.cpu().numpy()
    np.testing.assert_array_equal(b, A.values.sum(axis=1))  # ref: test_problem.py:60-68


def test_low_precision_copy_shares_structure():
    # ref: tests/test_problem.py:86-94
    from paper_2507_11512_b200.problem import to_low_precision
    A, _ = _single_rank_system(4, 4, 4)
    lo = to_low_precision(A)
    assert lo.values.dtype == np.float32 and lo.col_idx is A.col_idx
    np.testing.assert_array_equal(lo.values, A.values.astype(np.float32))


def test_matrix_market_output(tmp_path):
    # ref: tests/test_problem.py:109-120 -- 8^3 has 512 rows and 10,648 nonzeros
    from paper_2507_11512_b200.problem import write_matrix_market
    A, _ = _single_rank_system(8, 8, 8)
    path = tmp_path / "a.mtx"
    write_matrix_market(str(path), A, A.global_rows(), 512)
    lines = path.read_text().splitlines()
    assert lines[0] == "%%MatrixMarket matrix coordinate real general"
    assert lines[1] == "512 512 10648" and len(lines) == 2 + 10648
    assert lines[2] == "1 1 26"


def test_check_coloring_and_identity_coloring():
    # ref: tests/test_coloring.py:58-69
    from paper_2507_11512_b200.coloring import check_coloring, color, identity_coloring
    A, _ = _single_rank_system(4, 4, 4)
    assert check_coloring(A, color(A, "greedy"))
    ident = identity_coloring(64)
    assert ident.num_colors == 1 and list(ident.color_offsets) == [0, 64]
    assert not check_coloring(A, ident)


def test_permute_system_is_symmetric_permutation():
    # ref: tests/test_coloring.py:84-96: P A P^T with vectors permuted alike
    from paper_2507_11512_b200.coloring import color, permute_system
    A, vecs = _single_rank_system(4, 4, 4)
    c = color(A, "greedy")
    b = vecs.b.cpu().numpy()
    Ap, (bp,) = permute_system(A, [b], c)
    np.testing.assert_array_equal(bp, b[c.perm])
    dense = np.zeros((64, 64))
    densep = np.zeros((64, 64))
    for i in range(64):
        for s in range(A.row_nnz[i]):
            dense[i, A.col_idx[i, s]] = A.values[i, s]
        for s in range(Ap.row_nnz[i]):
            densep[i, Ap.col_idx[i, s]] = Ap.values[i, s]
    np.testing.assert_array_equal(densep, dense[np.ix_(c.perm, c.perm)])


# ---------------------------------------------------------------- krylov

def test_spmv_matches_sequential_oracle_bitwise():
    # ref: tests/test_krylov.py:33-40
    from paper_2507_11512_b200.krylov import spmv
    A, _ = _single_rank_system(4, 4, 4)
    x = np.zeros(A.n_cols_extended)
    x[:A.n_rows] = np.random.default_rng(3).integers(-9, 10, size=A.n_rows).astype(np.float64)
    y = spmv(A, x)
    assert isinstance(y, np.ndarray)
    np.testing.assert_array_equal(y, _seq_spmv(A.values, A.col_idx, x))


def test_cgs2_orthogonalizes_against_basis():
    # ref: tests/test_krylov.py:65-78 (host arrays, a private vector context)
    from paper_2507_11512_b200.krylov import cgs2_orthogonalize
    rng = np.random.default_rng(7)
    n, m = 64, 6
    Q = np.zeros((m + 1, n))
    Q[0] = rng.standard_normal(n)
    Q[0] /= np.linalg.norm(Q[0])
    H = np.zeros((m + 1, m))
    for k in range(4):
        w = rng.standard_normal(n)
        cgs2_orthogonalize(Q, k, w, H)
        assert np.max(np.abs(Q[:k + 1] @ w)) <= 1e-14 * np.linalg.norm(w)
        Q[k + 1] = w / np.linalg.norm(w)


def test_cgs2_coefficients_reproduce_projection():
    # ref: tests/test_krylov.py:81-93
    from paper_2507_11512_b200.krylov import cgs2_orthogonalize
    rng = np.random.default_rng(8)
    n = 32
    Q = np.zeros((3, n))
    Q[0] = rng.standard_normal(n)
    Q[0] /= np.linalg.norm(Q[0])
    w = rng.standard_normal(n)
    w_orig = w.copy()
    H = np.zeros((3, 2))
    h = cgs2_orthogonalize(Q, 0, w, H)
    assert np.allclose(w + h[0] * Q[0], w_orig, rtol=0.0, atol=1e-14)
    assert H[0, 0] == h[0]


def test_restarted_solve_converges():
    # ref: tests/test_krylov.py:145-155 -> 4 restarts, 18 iterations
    from paper_2507_11512_b200.krylov import gmres_solve
    from paper_2507_11512_b200.problem import to_low_precision
    A, _ = _single_rank_system(4, 4, 4)
    b = np.random.default_rng(42).standard_normal(A.n_rows)
    res = gmres_solve(A, to_low_precision(A), None, b, mode="double", tol=1e-10, m=5)
    assert res.converged and res.restarts == 4 and res.iterations == 18
    assert res.relres < 1e-10 and res.workspace is None


def test_solution_vector_matches_all_ones():
    # ref: tests/test_krylov.py:158-166 (x0 receives the solution in place)
    from paper_2507_11512_b200.krylov import gmres_solve
    from paper_2507_11512_b200.problem import to_low_precision
    A, vecs = _single_rank_system(4, 4, 4)
    x0 = np.zeros(A.n_cols_extended)
    res = gmres_solve(A, to_low_precision(A), None, vecs.b.cpu().numpy(), x0=x0, mode="double", tol=1e-12)
    assert res.converged
    assert np.allclose(x0[:A.n_rows], np.ones(A.n_rows), rtol=0.0, atol=1e-10)


def test_full_subspace_and_trivial_cases():
    # ref: tests/test_krylov.py:169-206
    from paper_2507_11512_b200.krylov import gmres_solve
    from paper_2507_11512_b200.problem import to_low_precision
    A, vecs = _single_rank_system(2, 2, 2)
    lo = to_low_precision(A)
    b = np.random.default_rng(7).standard_normal(8)
    res = gmres_solve(A, lo, None, b, mode="double", tol=1e-12, m=8)
    assert res.converged and res.restarts == 1 and res.iterations <= 8 and res.relres < 1e-12
    res = gmres_solve(A, lo, None, np.zeros(8), mode="double")
    assert res.converged and res.iterations == 0 and res.relres == 0.0
    x0 = np.ones(A.n_cols_extended)
    res = gmres_solve(A, lo, None, vecs.b.cpu().numpy(), x0=x0, mode="double")
    assert res.converged and res.iterations == 0 and res.relres == 0.0
    with pytest.raises(ValueError, match="unknown mode"):
        gmres_solve(A, lo, None, np.ones(8), mode="mxp")


def _preconditioned_solve(mode, m=30, keep_basis=False, tally=None):
    # ref: tests/test_krylov.py:209-218 (a user preconditioner calling h.apply)
    from paper_2507_11512_b200.krylov import gmres_solve
    hier = _hierarchy(16, 4)
    lv = hier.levels[0]
    b = lv.A_hi.values.sum(axis=1)

    def precond(r, tally=None):
        return hier.apply(r, tally=tally)

    res = gmres_solve(lv.A_hi, lv.A_lo, precond, b, mode=mode, tol=1e-9, m=m, keep_basis=keep_basis)
    hier.close()
    return res


def test_iteration_counts_and_workspace():
    # ref: tests/test_krylov.py:221-248
    res = _preconditioned_solve("double", keep_basis=True)
    assert res.converged and res.iterations == 16
    assert res.relres == pytest.approx(4.4911594142630304e-10, rel=1e-6)
    assert np.linalg.norm(res.workspace.Q[0]) == pytest.approx(1.0, rel=1e-12)
    res = _preconditioned_solve("mixed")
    assert res.converged and res.relres <= 1e-9 and abs(res.iterations - 20) <= 2
    res = _preconditioned_solve("double", m=8)
    assert res.converged and res.restarts >= 2 and len(res.boundary_pairs) == res.restarts
    assert all(a > 0.0 and b > 0.0 for a, b in res.boundary_pairs)


def test_solver_tally_covers_expected_motifs():
    # ref: tests/test_krylov.py:251-267
    from paper_2507_11512_b200.krylov import gmres_solve
    from paper_2507_11512_b200.metrics import Tally
    hier = _hierarchy(8, 4)
    lv = hier.levels[0]
    b = lv.A_hi.values.sum(axis=1)
    tally = Tally()
    res = gmres_solve(lv.A_hi, lv.A_lo, lambda r: hier.apply(r, tally=tally), b, tol=1e-9, tally=tally)
    assert res.converged
    for motif in ("SpMV", "GS", "Ortho", "Vector ops", "Restriction", "Prolongation"):
        assert tally.flops[motif] > 0 and tally.seconds[motif] > 0.0, motif
    hier.close()


# ---------------------------------------------------------------- smoother

def test_sweeps_match_sequential_oracle_bitwise():
    # ref: tests/test_smoother.py:27-48 (z mutated in place, host arrays)
    from paper_2507_11512_b200.smoother import forward_gs_sweep
    Ap, c = _permuted(4, 4, 4)
    r = np.random.default_rng(1).integers(-10, 11, size=Ap.n_rows).astype(float)
    z = np.zeros(Ap.n_cols_extended)
    z_ref = np.zeros(Ap.n_rows)
    forward_gs_sweep(Ap, r, z, c, z_is_zero=True)
    _seq_gs(Ap.values, Ap.col_idx, Ap.diag_pos, r, z_ref)
    np.testing.assert_array_equal(z[:Ap.n_rows], z_ref)
    forward_gs_sweep(Ap, r, z, c)
    _seq_gs(Ap.values, Ap.col_idx, Ap.diag_pos, r, z_ref)
    np.testing.assert_array_equal(z[:Ap.n_rows], z_ref)


def test_single_point_system_solved_exactly():
    # ref: tests/test_smoother.py:51-59
    from paper_2507_11512_b200.smoother import forward_gs_sweep
    Ap, c = _permuted(1, 1, 1)
    z = np.zeros(1)
    forward_gs_sweep(Ap, np.array([13.0]), z, c, z_is_zero=True)
    assert z[0] == 13.0 / 26.0


def test_three_sweep_residual_regression_on_8cubed():
    # ref: tests/test_smoother.py:62-81 -> relres 0.1973824330006174, decreasing norms
    from paper_2507_11512_b200.krylov import spmv
    from paper_2507_11512_b200.problem import generate_rhs
    from paper_2507_11512_b200.smoother import forward_gs_sweep
    Ap, c = _permuted(8, 8, 8)
    b = generate_rhs(Ap).b.cpu().numpy()
    z = np.zeros(Ap.n_cols_extended)
    norms = [np.linalg.norm(b)]
    for sweep in range(3):
        forward_gs_sweep(Ap, b, z, c, z_is_zero=(sweep == 0))
        norms.append(np.linalg.norm(b - spmv(Ap, z)))
    assert all(n1 < n0 for n0, n1 in zip(norms, norms[1:]))
    assert norms[-1] / norms[0] == pytest.approx(0.1973824330006174, rel=1e-12)


def test_low_high_precision_duality():
    # ref: tests/test_smoother.py:84-94
    from paper_2507_11512_b200.problem import to_low_precision
    from paper_2507_11512_b200.smoother import forward_gs_sweep
    Ap, c = _permuted(8, 8, 8)
    Al = to_low_precision(Ap)
    r = np.random.default_rng(2).integers(-10, 11, size=Ap.n_rows).astype(float)
    z_hi = np.zeros(Ap.n_cols_extended)
    z_lo = np.zeros(Al.n_cols_extended, dtype=np.float32)
    forward_gs_sweep(Ap, r, z_hi, c, z_is_zero=True)
    forward_gs_sweep(Al, r.astype(np.float32), z_lo, c, z_is_zero=True)
    assert np.linalg.norm(z_hi - z_lo.astype(np.float64)) / np.linalg.norm(z_hi) <= 1e-5


# ---------------------------------------------------------------- multigrid

def test_hierarchy_level_shapes():
    # ref: tests/test_multigrid.py:33-48
    h = _hierarchy(16, 4)
    assert [lv.domain.lnx for lv in h.levels] == [16, 8, 4, 2]
    assert [lv.A_hi.n_rows for lv in h.levels] == [4096, 512, 64, 8]
    assert h.levels[0].f2c is None
    assert [len(h.levels[i].f2c) for i in (1, 2, 3)] == [512, 64, 8]
    for lv in h.levels:
        assert lv.A_hi.values.dtype == np.float64 and lv.A_lo.values.dtype == np.float32
        assert lv.A_lo.col_idx is lv.A_hi.col_idx
    h.close()


def test_hierarchy_too_deep_raises():
    # ref: tests/test_multigrid.py:51-55
    from paper_2507_11512_b200.geometry import CoarseningError
    with pytest.raises(CoarseningError):
        _hierarchy(12, 4)


def test_f2c_matches_coordinate_doubling_and_is_unique():
    # ref: tests/test_multigrid.py:58-73
    h = _hierarchy(16, 4)
    for fine, coarse in zip(h.levels[:-1], h.levels[1:]):
        fg = fine.A_hi.col_global[np.arange(fine.A_hi.n_rows), fine.A_hi.diag_pos]
        cg = coarse.A_hi.col_global[np.arange(coarse.A_hi.n_rows), coarse.A_hi.diag_pos]
        f2c = np.asarray(coarse.f2c)
        assert len(np.unique(f2c)) == len(f2c)
        fd, cd = fine.domain, coarse.domain
        fx, fy, fz = fg[f2c] % fd.gnx, (fg[f2c] // fd.gnx) % fd.gny, fg[f2c] // (fd.gnx * fd.gny)
        cx, cy, cz = cg % cd.gnx, (cg // cd.gnx) % cd.gny, cg // (cd.gnx * cd.gny)
        assert np.array_equal(fx, 2 * cx) and np.array_equal(fy, 2 * cy) and np.array_equal(fz, 2 * cz)
    h.close()


def test_prolong_restrict_roundtrip_and_fused_restriction():
    # ref: tests/test_multigrid.py:76-104
    from paper_2507_11512_b200.krylov import spmv
    from paper_2507_11512_b200.multigrid import fused_residual_restrict, prolong_add, restrict_inject
    h = _hierarchy(8, 3)
    fine, coarse = h.levels[0], h.levels[1]
    rng = np.random.default_rng(11)
    x_c = rng.standard_normal(coarse.A_hi.n_rows)
    x_f = np.zeros(fine.A_hi.n_cols_extended)
    prolong_add(x_f, x_c, coarse.f2c)
    assert np.array_equal(restrict_inject(x_f, coarse.f2c), x_c)
    assert np.count_nonzero(x_f) == len(x_c)
    prolong_add(x_f, x_c, coarse.f2c)
    assert np.array_equal(restrict_inject(x_f, coarse.f2c), 2.0 * x_c)
    A = fine.A_hi
    rng = np.random.default_rng(5)
    x = np.zeros(A.n_cols_extended)
    x[:A.n_rows] = rng.standard_normal(A.n_rows)
    b = rng.standard_normal(A.n_rows)
    r_c = fused_residual_restrict(A, b, x, coarse.f2c)
    assert np.array_equal(r_c, restrict_inject(b - spmv(A, x), coarse.f2c))
    h.close()


def test_vcycle_exactness_linearity_and_precision():
    # ref: tests/test_multigrid.py:107-146
    from paper_2507_11512_b200.krylov import spmv
    h = _hierarchy(16, 4)
    rng = np.random.default_rng(0)
    r = rng.standard_normal(16 ** 3)
    z = h.apply(r).copy()
    assert np.array_equal(h.apply(2.0 * r), 2.0 * z)
    r1, r2 = rng.standard_normal(16 ** 3), rng.standard_normal(16 ** 3)
    za = h.apply(0.3 * r1 + 1.7 * r2).copy()
    zb = 0.3 * h.apply(r1).copy() + 1.7 * h.apply(r2).copy()
    assert np.linalg.norm(za - zb) <= 1e-12 * np.linalg.norm(za)
    z_lo = h.apply(r.astype(np.float32))
    assert z_lo.dtype == np.float32
    assert np.linalg.norm(z - z_lo.astype(np.float64)) / np.linalg.norm(z) <= 5e-7
    A = h.levels[0].A_hi
    b = A.values.sum(axis=1)
    x = np.zeros(A.n_cols_extended)
    x[:A.n_rows] = h.apply(b)
    assert np.linalg.norm(b - spmv(A, x)) / np.linalg.norm(b) < 0.5
    h.close()


def test_vcycle_tally_and_sweep_counts():
    # ref: tests/test_multigrid.py:149-185
    from paper_2507_11512_b200.metrics import Tally
    from paper_2507_11512_b200.smoother import SmootherWorkspace
    h = _hierarchy(8, 4)
    b = h.levels[0].A_hi.values.sum(axis=1)
    tally = Tally()
    h.apply(b, tally=tally)
    gs = sum(2 * 2 * lv.A_hi.nnz_total for lv in h.levels[:-1]) + 2 * h.levels[-1].A_hi.nnz_total
    restr = sum(int(np.sum(2 * f.A_hi.row_nnz[np.asarray(c.f2c)] + 1)) for f, c in zip(h.levels[:-1], h.levels[1:]))
    assert tally.flops["GS"] == gs and tally.flops["Restriction"] == restr
    assert tally.flops["Prolongation"] == sum(c.A_hi.n_rows for c in h.levels[1:])
    assert tally.flops["SpMV"] == tally.flops["Ortho"] == tally.flops["Vector ops"] == 0
    assert tally.seconds["GS"] > 0.0
    z_default = h.apply(b).copy()
    heavy = _hierarchy(8, 4, SmootherWorkspace(nu1=2, nu2=2, nu_c=3))
    t2 = Tally()
    z_heavy = heavy.apply(b, tally=t2)
    assert t2.flops["GS"] == sum(8 * lv.A_hi.nnz_total for lv in heavy.levels[:-1]) + \
        6 * heavy.levels[-1].A_hi.nnz_total
    assert not np.array_equal(z_heavy, z_default)
    h.close()
    heavy.close()


def test_vcycle_preconditioning_reduces_gmres_iterations():
    # ref: tests/test_multigrid.py:188-201 -> 10 preconditioned iterations at 8^3
    from paper_2507_11512_b200.krylov import gmres_solve
    h = _hierarchy(8, 4)
    lv = h.levels[0]
    b = lv.A_hi.values.sum(axis=1)
    res_pre = gmres_solve(lv.A_hi, lv.A_lo, lambda r, tally=None: h.apply(r, tally=tally), b, tol=1e-9)
    res_plain = gmres_solve(lv.A_hi, lv.A_lo, None, b, tol=1e-9)
    assert res_pre.converged and res_plain.converged
    assert res_pre.iterations == 10 and res_plain.iterations > res_pre.iterations
    h.close()
