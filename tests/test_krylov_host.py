"""Host-side GMRES pieces (CPU): the Givens update and the back substitution
keep the reference's semantics (ref: tests/test_krylov.py:96-132)."""
import numpy as np
import pytest

from paper_2507_11512_b200.krylov import BreakdownError, _back_substitute, givens_update


def test_givens_three_four_five():
    # ref: tests/test_krylov.py:96-111
    H = np.zeros((2, 1))
    H[0, 0], H[1, 0] = 3.0, 4.0
    t = np.zeros(2)
    t[0] = 10.0
    c, s = np.zeros(1), np.zeros(1)
    rec = givens_update(H, t, c, s, 0)
    assert H[0, 0] == 5.0 and H[1, 0] == 0.0
    assert c[0] == pytest.approx(0.6, rel=1e-15) and s[0] == pytest.approx(0.8, rel=1e-15)
    assert t[0] == pytest.approx(6.0, rel=1e-15) and t[1] == pytest.approx(-8.0, rel=1e-15)
    assert rec == pytest.approx(8.0, rel=1e-15)


def test_givens_fp32_storage_and_previous_rotations():
    """fp32 arrays: rotations computed in fp64 on promoted values, stored in fp32;
    the returned norm is read back from the stored entry (ref: krylov.py:132-159)."""
    H = np.zeros((3, 2), dtype=np.float32)
    H[:2, 0] = (3.0, 4.0)
    t = np.zeros(3, dtype=np.float32)
    t[0] = 10.0
    c, s = np.zeros(3, dtype=np.float32), np.zeros(3, dtype=np.float32)
    givens_update(H, t, c, s, 0)
    H[:3, 1] = (1.0, 2.0, 2.0)
    rec = givens_update(H, t, c, s, 1)
    col = np.array([1.0, 2.0, 2.0])
    top = 0.6 * col[0] + 0.8 * col[1]
    mid = -0.8 * col[0] + 0.6 * col[1]
    mu = np.hypot(mid, col[2])
    assert H.dtype == np.float32 and H[0, 1] == np.float32(top) and H[2, 1] == 0.0
    assert H[1, 1] == np.float32(mu)
    assert rec == abs(float(t[2])) and t.dtype == np.float32
    assert rec == pytest.approx(8.0 * col[2] / mu, rel=1e-6)


def test_givens_zero_column_raises():
    # ref: tests/test_krylov.py:114-119
    H = np.zeros((2, 1))
    t = np.zeros(2)
    t[0] = 1.0
    with pytest.raises(BreakdownError):
        givens_update(H, t, np.zeros(1), np.zeros(1), 0)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_back_substitute_matches_dense_solve(dtype):
    # ref: tests/test_krylov.py:122-132 (fp32 storage: solved on fp64 promotions)
    rng = np.random.default_rng(9)
    m = 8
    H = np.zeros((m + 1, m), dtype=dtype)
    R = np.triu(rng.standard_normal((m, m))) + 5.0 * np.eye(m)
    H[:m, :m] = R
    t = np.zeros(m + 1, dtype=dtype)
    t[:m] = rng.standard_normal(m)
    y = _back_substitute(H, t, m)
    y_ref = np.linalg.solve(H[:m, :m].astype(np.float64), t[:m].astype(np.float64))
    assert y.dtype == np.float64
    assert np.linalg.norm(y - y_ref) <= 1e-12 * np.linalg.norm(y_ref)
