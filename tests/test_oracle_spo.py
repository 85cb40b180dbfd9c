"""Pins of the NEXT-4 oracle (tricubic B-spline SPOs orc_spo_vgh and the
determinant ratio orc_det_ratio) against things other than itself:
partition of unity, scipy's 1D B-spline on separable tables, Marsden's
polynomial reproduction, finite differences, periodicity, and numpy's LU
determinant for the matrix determinant lemma (Eq. 6).
"""
import numpy as np
from scipy.interpolate import BSpline

import oracle
import qmcgen


def _pos(rng, M, L):
    return rng.random((M, 3)) * np.asarray(L)


def test_constant_table_is_constant():
    """Partition of unity: P = c everywhere -> v = c, grad = hess = 0."""
    T = np.full((5, 6, 7, 3), 0.75, np.float32)
    L = [2.0, 3.0, 4.0]
    v, g, h, _ = oracle.spo_vgh(T, 3, L, _pos(np.random.default_rng(1), 20, L))
    assert np.allclose(v, 0.75, rtol=0, atol=1e-15)
    assert np.abs(g).max() < 1e-13 and np.abs(h).max() < 1e-12


def _scipy_periodic_1d(c, n, L, x, nu=0):
    """1D periodic cubic B-spline of coefficients c[0..n-1] (control point j
    centred on node j) via scipy.interpolate.BSpline on the unwrapped sequence."""
    ce = np.asarray(c, dtype=np.float64)[(np.arange(n + 3) - 1) % n]
    spl = BSpline(np.arange(-3, n + 4, dtype=np.float64), ce, 3, extrapolate=False)
    u = np.mod(x, L) / L * n
    return spl(u, nu=nu) * (n / L) ** nu


def test_separable_table_matches_scipy_product():
    """P[ix][iy][iz][o] = A_o[ix] B_o[iy] C_o[iz]: v, grad and the Hessian are
    products of scipy 1D B-splines and their derivatives."""
    rng = np.random.default_rng(2)
    nx, ny, nz, no = 7, 5, 6, 4
    A, B, C = rng.normal(size=(no, nx)), rng.normal(size=(no, ny)), rng.normal(size=(no, nz))
    T = np.einsum("oi,oj,ok->ijko", A, B, C).astype(np.float32)
    # the oracle reads fp32 coefficients: use the rounded product as ground truth via a rank-1 check
    L = [1.7, 2.3, 3.1]
    pos = _pos(rng, 25, L)
    v, g, h, _ = oracle.spo_vgh(T, no, L, pos)
    for o in range(no):
        fx = [_scipy_periodic_1d(A[o], nx, L[0], pos[:, 0], nu) for nu in range(3)]
        fy = [_scipy_periodic_1d(B[o], ny, L[1], pos[:, 1], nu) for nu in range(3)]
        fz = [_scipy_periodic_1d(C[o], nz, L[2], pos[:, 2], nu) for nu in range(3)]
        ref_v = fx[0] * fy[0] * fz[0]
        ref_g = [fx[1] * fy[0] * fz[0], fx[0] * fy[1] * fz[0], fx[0] * fy[0] * fz[1]]
        ref_h = [fx[2] * fy[0] * fz[0], fx[1] * fy[1] * fz[0], fx[1] * fy[0] * fz[1],
                 fx[0] * fy[2] * fz[0], fx[0] * fy[1] * fz[1], fx[0] * fy[0] * fz[2]]
        scale = np.abs(A[o]).max() * np.abs(B[o]).max() * np.abs(C[o]).max()
        tol = 2e-7 * scale        # fp32 rounding of the product coefficients
        np.testing.assert_allclose(v[:, o], ref_v, atol=tol)
        for d in range(3):
            np.testing.assert_allclose(g[:, d, o], ref_g[d], atol=tol * 50)
        for q in range(6):
            np.testing.assert_allclose(h[:, q, o], ref_h[q], atol=tol * 2500)


def test_quadratic_reproduction_away_from_the_wrap():
    """Marsden: control values j^2 - 1/3 on node j reproduce u^2 (u = x n / L):
    v = u^2, dv/dx = 2u n/L, d2v/dx2 = 2 (n/L)^2, all y/z derivatives 0."""
    nx, ny, nz = 12, 4, 4
    j = np.arange(nx, dtype=np.float64)
    T = np.broadcast_to((j ** 2 - 1.0 / 3.0)[:, None, None, None], (nx, ny, nz, 1)).astype(np.float32).copy()
    L = [6.0, 1.0, 1.0]
    rng = np.random.default_rng(3)
    u = rng.uniform(1.0, nx - 2.0, 30)               # control points i-1..i+2 never wrap
    pos = np.stack([u * L[0] / nx, rng.random(30), rng.random(30)], 1)
    v, g, h, _ = oracle.spo_vgh(T, 1, L, pos)
    s = nx / L[0]
    np.testing.assert_allclose(v[:, 0], u ** 2, rtol=1e-6)          # fp32 control values
    np.testing.assert_allclose(g[:, 0, 0], 2 * u * s, rtol=1e-6)
    np.testing.assert_allclose(h[:, 0, 0], 2 * s * s, rtol=1e-5)
    assert np.abs(g[:, 1:, 0]).max() < 1e-9 and np.abs(h[:, 1:, 0]).max() < 1e-8


def test_gradient_hessian_vs_finite_differences():
    rng = np.random.default_rng(4)
    T = qmcgen.spo_table(4, 8, 9, 10, 5, 8)
    L = [3.0, 3.5, 4.0]
    pos = _pos(rng, 6, L)
    v, g, h, _ = oracle.spo_vgh(T, 5, L, pos)
    e = np.eye(3)
    hs = 1e-5
    pairs = [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]
    for m in range(6):
        f = lambda d: oracle.spo_vgh(T, 5, L, pos[m] + d)[0][0]   # noqa: E731
        for d in range(3):
            fd = (f(hs * e[d]) - f(-hs * e[d])) / (2 * hs)
            np.testing.assert_allclose(g[m, d], fd, atol=1e-6 * np.abs(g).max())
        for q, (a, b) in enumerate(pairs):
            hh = 1e-4
            fd = (f(hh * (e[a] + e[b])) - f(hh * (e[a] - e[b])) - f(hh * (e[b] - e[a])) + f(-hh * (e[a] + e[b]))) / (4 * hh * hh)
            np.testing.assert_allclose(h[m, q], fd, atol=1e-4 * np.abs(h).max())


def test_periodicity():
    rng = np.random.default_rng(5)
    T = qmcgen.spo_table(5, 6, 6, 6, 3)
    L = [2.0, 2.0, 2.0]
    pos = _pos(rng, 10, L)
    a = oracle.spo_vgh(T, 3, L, pos)
    for d in range(3):
        sh = np.zeros(3)
        sh[d] = L[d]
        b = oracle.spo_vgh(T, 3, L, pos + sh)
        c = oracle.spo_vgh(T, 3, L, pos - sh)
        for x, y, z in zip(a[:3], b[:3], c[:3]):
            np.testing.assert_allclose(x, y, atol=1e-12)
            np.testing.assert_allclose(x, z, atol=1e-12)


def test_determinant_lemma_against_lu_determinants():
    """rho = det(A')/det(A) with A(i,j) = phi_i(r_j) and column k replaced by
    phi(r'_k) (Eq. 6), by numpy's LU; G = grad ln det(A') and L = lap det(A')/det(A')
    by central differences of those determinants."""
    rng = np.random.default_rng(6)
    n = 12
    T = qmcgen.spo_table(6, 6, 7, 8, n)
    L = [3.0, 3.5, 4.0]
    R = _pos(rng, n, L)
    A = oracle.spo_vgh(T, n, L, R)[0].T                  # A[i][j] = phi_i(r_j)
    Ainv = np.linalg.inv(A)
    detA = np.linalg.det(A)

    def det_moved(k, r):
        Ap = A.copy()
        Ap[:, k] = oracle.spo_vgh(T, n, L, r)[0][0]
        return np.linalg.det(Ap)

    for k in (0, 5, 11):
        r = rng.random(3) * np.asarray(L)
        v, g, h, _ = oracle.spo_vgh(T, n, L, r)
        out, ab = oracle.det_ratio(Ainv[k:k + 1], v, g, h)
        rho = out[0, 0]
        assert abs(rho - det_moved(k, r) / detA) <= 1e-9 * max(1.0, ab[0, 0])
        hs = 1e-5
        e = np.eye(3)
        dm = det_moved(k, r)
        grad = np.array([(det_moved(k, r + hs * e[d]) - det_moved(k, r - hs * e[d])) / (2 * hs) for d in range(3)])
        np.testing.assert_allclose(out[0, 1:4], grad / dm, rtol=1e-5, atol=1e-6 * np.abs(grad / dm).max())
        hh = 1e-4
        lap = sum((det_moved(k, r + hh * e[d]) - 2 * dm + det_moved(k, r - hh * e[d])) / hh ** 2 for d in range(3))
        np.testing.assert_allclose(out[0, 4], lap / dm, rtol=1e-4, atol=1e-4 * abs(lap / dm))
    # a no-op move (r' = r_k): rho = 1 exactly up to the inverse's rounding
    for k in (2, 7):
        v, g, h, _ = oracle.spo_vgh(T, n, L, R[k])
        out, _ = oracle.det_ratio(Ainv[k:k + 1], v, g, h)
        assert abs(out[0, 0] - 1.0) < 1e-10
