"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Every oracle function is checked against: closed forms (Marsden's identity for
the cubic B-spline), an independent library routine (scipy.interpolate.BSpline),
brute force (27-image minimum image, O(N^2) pair sums written here in numpy),
finite differences, the worked examples printed in SPEC.md
(tests/golden/spec_examples.json) and invariances.  The independent references
below are written from the textbook definitions, not from oracle.c.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
from scipy.interpolate import BSpline

import oracle
import qmcgen

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ---------------------------------------------------------------------------
# Independent references (numpy / scipy), written from the definitions.
# ---------------------------------------------------------------------------
def ref_minimg_27(L, a, b):
    """Brute-force nearest image over the 27 shifts."""
    L = np.asarray(L, dtype=np.float64)
    a = np.atleast_2d(a).astype(np.float64)
    b = np.atleast_2d(b).astype(np.float64)
    best = None
    for sx in (-1, 0, 1):
        for sy in (-1, 0, 1):
            for sz in (-1, 0, 1):
                d = b - a + np.array([sx, sy, sz]) * L
                r = np.sqrt((d * d).sum(-1))
                if best is None:
                    best, bd = r, d
                else:
                    better = r < best
                    best = np.where(better, r, best)
                    bd = np.where(better[:, None], d, bd)
    return best, bd


def ref_functor(coef_channel, m, r_cut, r, nu=0):
    """scipy BSpline with uniform knots delta*(-3..m+3): the library cubic
    B-spline; zero at and beyond the cutoff."""
    delta = r_cut / m
    t = delta * np.arange(-3, m + 4, dtype=np.float64)
    spl = BSpline(t, np.asarray(coef_channel, dtype=np.float64), 3, extrapolate=False)
    r = np.asarray(r, dtype=np.float64)
    v = spl(r, nu=nu)
    return np.where(r < r_cut, v, 0.0)


def ref_j2_total(R1, N, n_up, fn):
    """sum_{i<j} U_s(|r_i - r_j|) in numpy + scipy (reading R1)."""
    tot = 0.0
    pos = R1[:, :N].T.astype(np.float64)
    for i in range(N):
        j = np.arange(i + 1, N)
        if j.size == 0:
            continue
        r, _ = ref_minimg_27(fn.L, np.repeat(pos[i:i + 1], j.size, 0), pos[j])
        same = (i < n_up) == (j < n_up)
        u = np.where(same, ref_functor(fn.coef[0], fn.m, fn.r_cut, r),
                     ref_functor(fn.coef[1], fn.m, fn.r_cut, r))
        tot += u.sum()
    return tot


def small_instance(N, W=4, seed=11, dtype=np.float64, P=1, mode="move", m=8):
    L = qmcgen.cell_length(N)
    Np = qmcgen.padded_size(N, 16)
    walkers = np.arange(W)
    R = qmcgen.positions(seed, walkers, N, Np, L, dtype)
    k = qmcgen.make_k(seed, W, N)
    rt = qmcgen.make_trials(seed, walkers, k, N, L, dtype, P=P, mode=mode)
    fn = qmcgen.make_functor(seed, L, m)
    return R, k, rt, fn


# ---------------------------------------------------------------------------
# Golden worked examples
# ---------------------------------------------------------------------------
def test_golden_min_image():
    for ex in GOLDEN["min_image"]:
        out = oracle.min_image(ex["L"], ex["a"], ex["b"])[0]
        assert out[0] == ex["dist"], ex["cite"]
        assert list(out[1:]) == ex["disp"], ex["cite"]


def test_golden_stage_candidate_row_N2():
    ex = GOLDEN["stage_candidate_row"][0]
    # N = 2: particle 0 moved to r0_new; the row entry for particle 1 is 5.
    R = np.zeros((1, 3, 16))
    R[0, :, 0] = [1.0, 1.0, 1.0]
    R[0, :, 1] = ex["r1"]
    fn = qmcgen.Functor(L=tuple(ex["L"]), r_cut=ex["L"][0] / 2, m=8, coef=np.zeros((2, 11)))
    rt = np.array(ex["r0_new"], dtype=np.float64).reshape(1, 1, 3)
    _, _, row = oracle.eval_j2(R, np.array([0]), rt, fn, n_total=2, n_up=1, row=True)
    assert row[0, 0, 0, 1] == ex["temp1"], ex["cite"]


def test_golden_functor_examples():
    for ex in GOLDEN["functor_eval_vgl"]:
        c = np.full(ex["m"] + 3, ex["c"])
        out = oracle.bspline(c, ex["m"], ex["r_cut"], [ex["r"]])[0]
        np.testing.assert_allclose(out, ex["out"], atol=1e-14, err_msg=ex["cite"])


def test_golden_padded_size():
    for ex in GOLDEN["padded_size"]:
        assert qmcgen.padded_size(ex["n"], ex["block"]) == ex["out"], ex["cite"]
    with pytest.raises(ValueError):
        qmcgen.padded_size(5, 0)


def test_golden_storage_laws():
    a, b, c = GOLDEN["storage_laws"]
    assert a["N"] * (a["N"] - 1) // 2 == a["packed"], a["cite"]
    assert b["N"] * qmcgen.padded_size(b["N"], b["block"]) == b["padded"], b["cite"]
    assert 5 * c["N"] ** 2 * 8 == c["ref_j2_bytes_double"], c["cite"]
    assert 5 * c["N"] == c["opt_j2_scalars"], c["cite"]


# ---------------------------------------------------------------------------
# Functor pins
# ---------------------------------------------------------------------------
M, RC = 8, 3.7
DELTA = RC / M
RS = np.linspace(0.0, RC * (1 - 1e-9), 977)


def _knots():
    return (np.arange(M + 3) - 1) * DELTA  # x_j = (j - 1) delta


def test_bspline_constant_partition_of_unity():
    out = oracle.bspline(np.full(M + 3, 0.625), M, RC, RS)
    np.testing.assert_allclose(out[:, 0], 0.625, rtol=0, atol=1e-15)
    np.testing.assert_allclose(out[:, 1:], 0.0, atol=1e-13)


def test_bspline_linear_precision():
    x = _knots()
    out = oracle.bspline(0.3 + 1.7 * x, M, RC, RS)
    np.testing.assert_allclose(out[:, 0], 0.3 + 1.7 * RS, rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(out[:, 1], 1.7, rtol=1e-13)
    np.testing.assert_allclose(out[:, 2], 0.0, atol=1e-11)


def test_bspline_quadratic_closed_form():
    x = _knots()
    out = oracle.bspline(x ** 2 - DELTA ** 2 / 3, M, RC, RS)
    np.testing.assert_allclose(out[:, 0], RS ** 2, rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(out[:, 1], 2 * RS, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(out[:, 2], 2.0, rtol=1e-11)


def test_bspline_cubic_closed_form():
    x = _knots()
    out = oracle.bspline(x ** 3 - x * DELTA ** 2, M, RC, RS)
    np.testing.assert_allclose(out[:, 0], RS ** 3, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(out[:, 1], 3 * RS ** 2, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(out[:, 2], 6 * RS, rtol=1e-10, atol=1e-11)


def test_bspline_matches_scipy_library():
    rng = np.random.default_rng(5)
    for m in (4, 8, 13, 64):
        c = rng.normal(size=m + 3)
        rc = 2.5
        r = np.concatenate([rng.random(500) * rc, np.arange(m) * rc / m])  # include knots
        out = oracle.bspline(c, m, rc, r)
        for nu in range(3):
            ref = ref_functor(c, m, rc, r, nu)
            np.testing.assert_allclose(out[:, nu], ref, rtol=1e-11,
                                       atol=1e-12 * (m / rc) ** nu)


def test_bspline_finite_differences():
    rng = np.random.default_rng(6)
    c = rng.random(M + 3)
    r = DELTA * 0.1 + rng.random(300) * (RC - 0.2 * DELTA)
    h = 1e-5
    up, dn = oracle.bspline(c, M, RC, r + h), oracle.bspline(c, M, RC, r - h)
    mid = oracle.bspline(c, M, RC, r)
    fd1 = (up[:, 0] - dn[:, 0]) / (2 * h)
    fd2 = (up[:, 1] - dn[:, 1]) / (2 * h)
    scale1 = np.abs(c).max() / DELTA
    scale2 = np.abs(c).max() / DELTA ** 2
    assert np.max(np.abs(fd1 - mid[:, 1])) / scale1 < 1e-6
    assert np.max(np.abs(fd2 - mid[:, 2])) / scale2 < 1e-5


def test_bspline_c2_zero_at_cutoff_and_beyond():
    rng = np.random.default_rng(7)
    c = np.concatenate([rng.random(M), np.zeros(3)])
    near = oracle.bspline(c, M, RC, [RC * (1 - 1e-7)])[0]
    assert abs(near[0]) < 1e-18 and abs(near[1]) < 1e-12 and abs(near[2]) < 1e-5
    far = oracle.bspline(c, M, RC, [RC, RC * 1.5, 1e30])
    assert np.all(far == 0.0)


# ---------------------------------------------------------------------------
# Minimum image pins
# ---------------------------------------------------------------------------
def test_min_image_vs_27_image_brute_force():
    rng = np.random.default_rng(8)
    L = np.array([7.0, 9.5, 11.25])
    a = rng.random((1000, 3)) * L
    b = rng.random((1000, 3)) * L
    out = oracle.min_image(L, a, b)
    r, d = ref_minimg_27(L, a, b)
    np.testing.assert_allclose(out[:, 0], r, rtol=1e-12)
    np.testing.assert_allclose(out[:, 1:], d, atol=1e-12)
    assert np.all(out[:, 1:] > -L / 2) and np.all(out[:, 1:] <= L / 2)


def test_min_image_exact_for_fp32_inputs():
    """fp32 coordinates in [0, L) with fp32 L: the fp64 oracle displacement is
    the exact real min-image displacement (checked with rationals)."""
    rng = np.random.default_rng(9)
    L = np.float32(85.0132)
    a = (rng.random((200, 3)) * L).astype(np.float32)
    b = (rng.random((200, 3)) * L).astype(np.float32)
    out = oracle.min_image([float(L)] * 3, a, b)
    FL = Fraction(float(L))
    for n in range(200):
        for c in range(3):
            t = Fraction(float(b[n, c])) - Fraction(float(a[n, c]))
            if t > FL / 2:
                t -= FL
            elif t <= -FL / 2:
                t += FL
            assert Fraction(out[n, 1 + c]) == t


# ---------------------------------------------------------------------------
# Hot-path (eval) pins
# ---------------------------------------------------------------------------
def test_eval_N2_is_single_functor_value():
    R, k, rt, fn = small_instance(2, W=16, seed=3)
    out, _, _ = oracle.eval_j2(R, k, rt, fn, n_total=2, n_up=1)
    for w in range(16):
        other = 1 - k[w]
        r, d = ref_minimg_27(fn.L, rt[w, 0], R[w, :, other])
        ch = 0 if (other < 1) == (k[w] < 1) else 1   # always opposite for N=2
        assert ch == 1
        u = [ref_functor(fn.coef[ch], fn.m, fn.r_cut, r, nu)[0] for nu in range(3)]
        exp = [u[0], *(-u[1] * d[0] / r[0]), u[2] + 2 * u[1] / r[0]]
        np.testing.assert_allclose(out[w, 0], exp, rtol=1e-12, atol=1e-13)


def test_eval_beyond_cutoff_contributes_exactly_zero():
    L = 10.0
    fn = qmcgen.make_functor(1, L)
    R = np.zeros((1, 3, 16))
    R[0, :, 0] = [1.0, 1.0, 1.0]
    R[0, :, 1] = [6.5, 6.5, 1.0]       # distance 7.78 > r_cut = 5
    rt = np.array([[[1.0, 1.0, 1.0]]])
    out, absout, _ = oracle.eval_j2(R, np.array([0]), rt, fn, n_total=2, n_up=1)
    assert np.all(out == 0.0) and np.all(absout == 0.0)


@pytest.mark.parametrize("N", [3, 14, 33, 64])
def test_delta_j2_equals_brute_force_pair_sum(N):
    """Eq. (5) vs Eq. (3): V(r'_k) - V(r_k) == J2(R') - J2(R) (reading R1)."""
    W = 6
    R, k, rt, fn = small_instance(N, W=W, seed=20 + N, P=2, mode="drift")
    out, _, _ = oracle.eval_j2(R, k, rt, fn, n_total=N, n_up=N // 2)
    for w in range(W):
        Rp = R[w].copy()
        Rp[:, k[w]] = rt[w, 1]
        dj_brute = ref_j2_total(Rp, N, N // 2, fn) - ref_j2_total(R[w], N, N // 2, fn)
        dj_orc = out[w, 1, 0] - out[w, 0, 0]
        scale = max(1.0, abs(ref_j2_total(R[w], N, N // 2, fn)))
        assert abs(dj_orc - dj_brute) <= 1e-12 * scale
        # the oracle's own brute-force entry point agrees with the numpy one
        assert abs(oracle.j2_total(R[w], N, N // 2, fn) - ref_j2_total(R[w], N, N // 2, fn)) <= 1e-12 * scale


def test_gradient_and_laplacian_vs_finite_differences():
    """G = grad_{r'} V, L = lap_{r'} V (Alg. 1 L8; reading R12)."""
    N, W = 40, 5
    R, k, rt, fn = small_instance(N, W=W, seed=31)
    out, absout, _ = oracle.eval_j2(R, k, rt, fn, n_total=N, n_up=N // 2)
    h1, h2 = 1e-5 * fn.L[0], 1e-4 * fn.L[0]
    for w in range(W):
        base = rt[w:w + 1]
        def V(shift):
            t = (base + shift).reshape(1, 1, 3)
            return oracle.eval_j2(R[w:w + 1], k[w:w + 1], t, fn, n_total=N, n_up=N // 2)[0][0, 0, 0]
        g = np.array([(V(h1 * e) - V(-h1 * e)) / (2 * h1) for e in np.eye(3)])
        lap = sum((V(h2 * e) - 2 * V(0 * e) + V(-h2 * e)) / h2 ** 2 for e in np.eye(3))
        assert np.max(np.abs(g - out[w, 0, 1:4])) <= 1e-6 * max(absout[w, 0, 1:4].max(), 1)
        assert abs(lap - out[w, 0, 4]) <= 1e-5 * max(absout[w, 0, 4], 1)


def test_symmetric_pairs_give_zero_gradient():
    L = 12.0
    fn = qmcgen.make_functor(4, L)
    rng = np.random.default_rng(12)
    c = np.array([L / 2] * 3)
    v = (rng.random((10, 3)) - 0.5) * 5.0
    src = np.concatenate([c + v, c - v])            # 20 sources in +/- pairs
    # all sources in the same spin half as k: put k last (index 20), n_up = 21
    R = np.zeros((1, 3, 32))
    R[0, :, :20] = src.T
    R[0, :, 20] = c
    out, absout, _ = oracle.eval_j2(R, np.array([20]), c.reshape(1, 1, 3), fn,
                                    n_total=21, n_up=21)
    assert np.all(np.abs(out[0, 0, 1:4]) <= 1e-14 * max(1.0, absout[0, 0, 1:4].max()))
    assert out[0, 0, 0] != 0.0


def test_quadratic_functor_integer_laplacian():
    """With U = r^2 (quadratic coefficient sequence, SURVEY 8(c) pin (iii)):
    V = sum r_i^2, G = -2 sum d_i, L = 6 * (number of in-cutoff sources)."""
    N, W = 300, 8
    R, k, rt, fn = small_instance(N, W=W, seed=41)
    x = (np.arange(fn.m + 3) - 1) * fn.delta
    q = np.stack([x ** 2 - fn.delta ** 2 / 3] * 2)
    fq = qmcgen.Functor(L=fn.L, r_cut=fn.r_cut, m=fn.m, coef=q)
    out, _, _ = oracle.eval_j2(R, k, rt, fq, n_total=N, n_up=N // 2)
    for w in range(W):
        i = np.array([j for j in range(N) if j != k[w]])
        r, d = ref_minimg_27(fn.L, np.repeat(rt[w, :1], i.size, 0), R[w, :, i])
        inside = r < fn.r_cut
        n_in = int(inside.sum())
        assert abs(out[w, 0, 4] - 6 * n_in) <= 1e-10 * n_in
        np.testing.assert_allclose(out[w, 0, 0], (r[inside] ** 2).sum(), rtol=1e-12)
        np.testing.assert_allclose(out[w, 0, 1:4], -2 * d[inside].sum(0), atol=1e-10 * n_in)


def test_noop_move_gives_bitwise_zero_delta():
    R, k, rt, fn = small_instance(50, W=8, seed=51, P=2, mode="noop")
    out, _, _ = oracle.eval_j2(R, k, rt, fn, n_total=50, n_up=25)
    assert np.array_equal(out[:, 0], out[:, 1])


def test_translation_and_permutation_invariance():
    N, W = 120, 4
    R, k, rt, fn = small_instance(N, W=W, seed=61)
    out, absout, _ = oracle.eval_j2(R, k, rt, fn, n_total=N, n_up=N // 2)
    L = fn.L[0]
    shift = np.array([1.234, -4.5, 2.75])
    R2 = np.mod(R + shift.reshape(1, 3, 1), L)
    R2[:, :, N:] = 0
    rt2 = np.mod(rt + shift, L)
    out2, _, _ = oracle.eval_j2(R2, k, rt2, fn, n_total=N, n_up=N // 2)
    assert np.max(oracle.normalized_error(out2, out, absout, fn)) < 1e-12
    # permute sources within each spin half (k's slot moves with it)
    rng = np.random.default_rng(62)
    perm = np.concatenate([rng.permutation(N // 2), N // 2 + rng.permutation(N - N // 2)])
    R3 = R.copy()
    R3[:, :, :N] = R[:, :, perm]
    inv = np.argsort(perm)
    k3 = inv[k].astype(np.int32)
    out3, _, _ = oracle.eval_j2(R3, k3, rt, fn, n_total=N, n_up=N // 2)
    assert np.max(oracle.normalized_error(out3, out, absout, fn)) < 1e-12


def test_sharded_partial_sums_equal_unsplit():
    N, W = 203, 6
    R, k, rt, fn = small_instance(N, W=W, seed=71)
    out, absout, _ = oracle.eval_j2(R, k, rt, fn, n_total=N, n_up=N // 2)
    cuts = [0, 37, 101, 150, N]
    tot = np.zeros_like(out)
    for a, b in zip(cuts[:-1], cuts[1:]):
        Rs = np.zeros((W, 3, 128))
        Rs[:, :, :b - a] = R[:, :, a:b]
        part, _, _ = oracle.eval_j2(Rs, k, rt, fn, n_total=N, n_up=N // 2,
                                    i_offset=a, n_local=b - a)
        tot += part
    assert np.max(oracle.normalized_error(tot, out, absout, fn)) < 1e-13


def test_row_output_matches_brute_force():
    N, W = 70, 3
    R, k, rt, fn = small_instance(N, W=W, seed=81, dtype=np.float32)
    _, _, row = oracle.eval_j2(R, k, rt, fn, n_total=N, n_up=N // 2, row=True)
    for w in range(W):
        i = np.array([j for j in range(N) if j != k[w]])
        r, d = ref_minimg_27(fn.L, np.repeat(rt[w, :1].astype(np.float64), i.size, 0),
                             R[w, :, i].astype(np.float64))
        np.testing.assert_allclose(row[w, 0, 0, i], r, rtol=1e-15)
        np.testing.assert_array_equal(row[w, 0, 1:, i], d)   # exact for fp32 inputs
        assert np.isnan(row[w, 0, 0, k[w]])                  # slot k untouched


def test_coincident_source_is_refused():
    R, k, rt, fn = small_instance(10, W=2, seed=91, mode="noop")
    k2 = k.copy()
    k2[0] = (k[0] + 1) % 10            # the trial sits on a source that is now counted
    with pytest.raises(oracle.CoincidentError):
        oracle.eval_j2(R, k2, rt, fn, n_total=10, n_up=5)


def test_threads_do_not_change_result():
    R, k, rt, fn = small_instance(90, W=13, seed=95)
    a = oracle.eval_j2(R, k, rt, fn, n_total=90, n_up=45, threads=1)[0]
    b = oracle.eval_j2(R, k, rt, fn, n_total=90, n_up=45, threads=5)[0]
    assert np.array_equal(a, b)


def test_min_image_tie_range_is_half_open():
    """disp_d in (-L_d/2, L_d/2] (reading R7): exact ties map to +L/2."""
    L = [10.0, 10.0, 10.0]
    out = oracle.min_image(L, [[5.0, 0.0, 0.0], [0.0, 0.0, 0.0]], [[0.0, 0.0, 0.0], [5.0, 0.0, 0.0]])
    assert out[0, 1] == 5.0 and out[1, 1] == 5.0


# ---------------------------------------------------------------------------
# NEXT-1: one-body Jastrow over the AB row
# ---------------------------------------------------------------------------
def _j1_instance(n_ions, W, seed, P=1, mode="move", N=40):
    L = qmcgen.cell_length(max(N, 12 * n_ions))
    fn1 = qmcgen.make_j1_functor(seed, L)
    ions, start = qmcgen.make_ions(seed, n_ions, qmcgen.padded_size(n_ions, 16), L, np.float64)
    R = qmcgen.positions(seed, np.arange(W), N, qmcgen.padded_size(N, 16), L, np.float64)
    k = qmcgen.make_k(seed, W, N)
    rt = qmcgen.make_trials(seed, np.arange(W), k, N, L, np.float64, P=P, mode=mode)
    return L, fn1, ions, start, R, k, rt


def _ref_j1_point(fn1, ions, start, r):
    """sum_I U_s(|r_I - r|) with scipy B-splines and 27-image distances."""
    tot = 0.0
    for s in range(len(fn1.m)):
        idx = np.arange(start[s], start[s + 1])
        if idx.size == 0:
            continue
        rr, _ = ref_minimg_27(fn1.L, np.repeat(np.asarray(r, float)[None], idx.size, 0), ions[:, idx].T)
        tot += ref_functor(fn1.coef[s, :fn1.m[s] + 3], fn1.m[s], fn1.r_cut[s], rr).sum()
    return tot


def test_j1_single_ion_is_the_functor():
    L, fn1, _, _, _, _, _ = _j1_instance(4, 1, seed=3)
    rng = np.random.default_rng(0)
    for s in range(2):
        ion = np.zeros((3, 16))
        ion[:, 0] = [L / 2, L / 2, L / 2]
        start = np.array([0, 1, 1]) if s == 0 else np.array([0, 0, 1])
        for _ in range(20):
            r = ion[:, 0] + (rng.random(3) - 0.5) * fn1.r_cut[s]
            out, _ = oracle.eval_j1(ion, start, r.reshape(1, 1, 3), fn1)
            d = ion[:, 0] - r
            rho = np.linalg.norm(d)
            c = fn1.coef[s, :fn1.m[s] + 3]
            u = [ref_functor(c, fn1.m[s], fn1.r_cut[s], rho, nu) for nu in range(3)]
            exp = [u[0], *(-u[1] * d / rho), u[2] + 2 * u[1] / rho]
            np.testing.assert_allclose(out[0, 0], exp, rtol=1e-11, atol=1e-12)
            # G points along +-(r - r_I) (radial symmetry)
            assert np.linalg.norm(np.cross(out[0, 0, 1:4], r - ion[:, 0])) <= 1e-9 * max(1, np.abs(out[0, 0, 1:4]).max())


def test_j1_per_species_cutoff():
    L, fn1, _, _, _, _, _ = _j1_instance(4, 1, seed=3)
    assert fn1.r_cut[1] < fn1.r_cut[0]
    ion = np.zeros((3, 16))
    ion[:, 0] = [L / 2] * 3
    r = ion[:, 0] + np.array([0.5 * (fn1.r_cut[0] + fn1.r_cut[1]), 0, 0])   # inside U_0, beyond U_1
    out0, _ = oracle.eval_j1(ion, np.array([0, 1, 1]), r.reshape(1, 1, 3), fn1)
    out1, _ = oracle.eval_j1(ion, np.array([0, 0, 1]), r.reshape(1, 1, 3), fn1)
    assert out0[0, 0, 0] != 0.0 and np.all(out1 == 0.0)


@pytest.mark.parametrize("n_ions", [1, 5, 32])
def test_delta_j1_equals_brute_force(n_ions):
    """Delta J1 = J1(R') - J1(R) with J1 = sum_i sum_I U_I(|r_I - r_i|)
    (Eq. 3 first term) equals U^1_k(R') - U^1_k(R)."""
    N, W = 30, 4
    L, fn1, ions, start, R, k, rt = _j1_instance(n_ions, W, seed=10 + n_ions, P=2, mode="drift", N=N)
    out, _ = oracle.eval_j1(ions, start, rt, fn1)
    for w in range(W):
        J = lambda Rw: sum(_ref_j1_point(fn1, ions, start, Rw[:, i]) for i in range(N))  # noqa: E731
        Rp = R[w].copy()
        Rp[:, k[w]] = rt[w, 1]
        dj = J(Rp) - J(R[w])
        assert abs((out[w, 1, 0] - out[w, 0, 0]) - dj) <= 1e-12 * max(1.0, abs(J(R[w])))


def test_j1_gradient_laplacian_fd():
    L, fn1, ions, start, _, _, rt = _j1_instance(24, 4, seed=21, N=288)
    out, absout = oracle.eval_j1(ions, start, rt, fn1)
    h1, h2 = 1e-5 * L, 1e-4 * L
    for w in range(4):
        V = lambda sh: oracle.eval_j1(ions, start, (rt[w, 0] + sh).reshape(1, 1, 3), fn1)[0][0, 0, 0]  # noqa: E731
        g = np.array([(V(h1 * e) - V(-h1 * e)) / (2 * h1) for e in np.eye(3)])
        lap = sum((V(h2 * e) - 2 * V(0 * e) + V(-h2 * e)) / h2 ** 2 for e in np.eye(3))
        assert np.max(np.abs(g - out[w, 0, 1:4])) <= 1e-6 * max(absout[w, 0, 1:4].max(), 1)
        assert abs(lap - out[w, 0, 4]) <= 1e-5 * max(absout[w, 0, 4], 1)
