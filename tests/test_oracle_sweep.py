"""Pins of the sweep oracle (oracle/oracle.c orc_propose_f32, orc_sweep) against
things other than itself: exact rational arithmetic for the fp32 proposal, the
numpy+scipy brute-force pair sum J2 = sum_{i<j} U (reading R1) for every
move's Delta J2, the from-scratch state of the final configuration, and the
scipy functor for Delta J1.

PAPER:842-851 (Alg. 1 L4-L9: the particle-by-particle sweep)
(Eq. 4-5: the ratio e^{Delta J1 + Delta J2}), PAPER:1382-1393 (Delta J2 =
U^2_k(R') - U^2_k(R) with U^2_k(R) held in the 5N state)
(Delta J1).
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import qmcgen
from test_oracle_pins import ref_functor, ref_j2_total


def _f32_ulp(x):
    x = np.float32(x)
    return float(np.nextafter(x, np.float32(np.inf)) - x)


def test_propose_is_the_wrapped_sum():
    """r' in [0, L) and r' == r + delta (mod L) to within one fp32 rounding
    (exact rationals); delta = 0 returns r bitwise; no wrap -> the correctly
    rounded sum."""
    rng = np.random.default_rng(1)
    L = qmcgen.cell_length(768)
    n = 4000
    r = (rng.random((n, 3)) * L).astype(np.float32)
    r = np.where(r >= np.float32(L), np.float32(0), r)
    d = rng.normal(0.0, 0.1, (n, 3)).astype(np.float32)
    # boundary cases: just below L pushed up, 0 pushed down by a tiny amount, exact multiples
    r[:6] = np.float32(np.nextafter(np.float32(L), np.float32(0)))
    d[:3] = np.float32(1e-7)
    d[3:6] = np.float32(0.0)
    r[6:12] = np.float32(0.0)
    d[6:9] = np.float32(-1e-9)
    d[9:12] = np.float32(-0.3)
    out = oracle.propose_f32((L, L, L), r, d)
    Lf = np.float32(L)
    assert np.all(out >= 0) and np.all(out < Lf)
    LF = Fraction(float(Lf))
    for i in range(n):
        for c in range(3):
            exact = (Fraction(float(r[i, c])) + Fraction(float(d[i, c]))) % LF
            err = abs(Fraction(float(out[i, c])) - exact)
            err = min(err, LF - err)            # distance on the circle
            assert err <= Fraction(_f32_ulp(Lf)), (i, c)
    z = oracle.propose_f32((L, L, L), r, np.zeros_like(d))
    assert np.array_equal(z, r)
    inside = (r.astype(np.float64) + d.astype(np.float64) >= 0) & (r.astype(np.float64) + d.astype(np.float64) < float(Lf) - 1e-3)
    exact_sum = np.array([[float(np.float32(Fraction(float(a)) + Fraction(float(b))))
                           for a, b in zip(ra, da)] for ra, da in zip(r[:200], d[:200])])
    assert np.array_equal(out[:200][inside[:200]], exact_sum[inside[:200]].astype(np.float32))


def _instance(N, W, seed, S, order):
    L = qmcgen.cell_length(N)
    Np = qmcgen.padded_size(N, 32)
    R = qmcgen.positions(seed, np.arange(W), N, Np, L, np.float32)
    fn = qmcgen.make_functor(seed, L)
    ks, delta, u = qmcgen.make_sweep_moves(seed, W, N, S, order=order)
    state = np.stack([oracle.j2_state(R[w], N, N // 2, fn)[0] for w in range(W)])
    return R, fn, ks, delta, u, state, L


@pytest.mark.parametrize("N,order,sweeps", [(14, "ordered", 3), (33, "random", 2), (9, "random", 4)])
def test_sweep_delta_j2_is_the_brute_force_pair_sum_difference(N, order, sweeps):
    """Every move's dJ2 (ratio from the stored state) equals J2(R') - J2(R) of
    the brute-force numpy+scipy pair sum (reading R1) with r'_k = the wrapped
    proposal from the walker's current r_k -- over several sweeps and with
    repeated k; the decisions are u < exp(2 dJ2); R evolves exactly by the
    accepted proposals."""
    W = 2
    S = sweeps * N
    R, fn, ks, delta, u, state, L = _instance(N, W, 400 + N, S, order)
    R2, S2, acc, dj, _ = oracle.sweep(R, state, ks, delta, u, fn, N, N // 2)
    Rx = R.astype(np.float32).copy()
    for s in range(S):
        for w in range(W):
            k = ks[s, w]
            rn = oracle.propose_f32((L, L, L), Rx[w, :, k], delta[s, w])[0]
            Rp = Rx[w].copy()
            Rp[:, k] = rn
            j_old = ref_j2_total(Rx[w].astype(np.float64), N, N // 2, fn)
            j_new = ref_j2_total(Rp.astype(np.float64), N, N // 2, fn)
            assert abs(dj[s, w] - (j_new - j_old)) <= 1e-10 * max(1.0, abs(j_old)), (s, w)
            assert acc[s, w] == int(u[s, w] < np.exp(dj[s, w]) ** 2)
            if acc[s, w]:
                Rx[w] = Rp
    assert np.array_equal(R2, Rx)
    assert 0 < acc.sum() < acc.size
    for w in range(W):
        fresh, ab = oracle.j2_state(R2[w].astype(np.float64), N, N // 2, fn)
        assert oracle.normalized_error_state(S2[w], fresh, ab, fn).max() <= 1e-11


def test_sweep_forced_decisions_and_invalid_k():
    """forced decisions drive the trajectory (the oracle still reports its own);
    a move with k outside [0, N) changes nothing and reports -1."""
    N, W, S = 20, 3, 40
    R, fn, ks, delta, u, state, L = _instance(N, W, 77, S, "random")
    _, _, own, _, _ = oracle.sweep(R, state, ks, delta, u, fn, N, N // 2)
    forced = 1 - own
    R2, S2, acc2, dj2, _ = oracle.sweep(R, state, ks, delta, u, fn, N, N // 2, forced=forced)
    assert acc2[0].tolist() == own[0].tolist()          # first move: same state, same decision
    # replaying the forced decisions by hand gives the same final configuration
    Rx = R.copy()
    for s in range(S):
        for w in range(W):
            if forced[s, w]:
                Rx[w, :, ks[s, w]] = oracle.propose_f32((L, L, L), Rx[w, :, ks[s, w]], delta[s, w])[0]
    assert np.array_equal(R2, Rx)
    ks_bad = ks.copy()
    ks_bad[5, 1] = N
    ks_bad[9, 2] = -3
    R3, S3, acc3, dj3, _ = oracle.sweep(R, state, ks_bad, delta, u, fn, N, N // 2,
                                        forced=np.where(ks_bad >= 0, own, 1))
    assert acc3[5, 1] == -1 and acc3[9, 2] == -1 and dj3[5, 1] == 0.0


def _ref_j1(ions, start, fn1, r):
    """U^1 at r: sum over ions of the scipy functor of the ion's species at the
    27-image distance."""
    from test_oracle_pins import ref_minimg_27
    tot = 0.0
    for s in range(len(fn1.m)):
        a, b = int(start[s]), int(start[s + 1])
        if b <= a:
            continue
        d, _ = ref_minimg_27(fn1.L, np.repeat(np.asarray(r, np.float64)[None], b - a, 0), ions[:, a:b].T)
        tot += ref_functor(fn1.coef[s][:fn1.m[s] + 3], fn1.m[s], fn1.r_cut[s], d).sum()
    return tot


def test_sweep_with_j1_adds_delta_j1_and_writes_the_row():
    """With ions: dJ = dJ2 + dJ1, dJ1 = U^1(r'_k) - U^1(r_k) by the scipy
    functor (Eq. 4); accepted electrons' J1 rows equal the J1
    oracle at their final positions (eval_j1, pinned in test_oracle_pins)."""
    N, W, S, n_ions = 24, 2, 48, 10
    R, fn, ks, delta, u, state, L = _instance(N, W, 91, S, "random")
    ions, start = qmcgen.make_ions(91, n_ions, 16, L, np.float64, n_species=2)
    fn1 = qmcgen.make_j1_functor(91, L, n_species=2)
    s_j1 = np.zeros((W, 5, R.shape[2]))
    R2, S2, acc, dj, S1 = oracle.sweep(R, state, ks, delta, u, fn, N, N // 2, j1=(ions, start, fn1, s_j1))
    _, _, _, dj2only, _ = oracle.sweep(R, state, ks, delta, u, fn, N, N // 2, forced=acc)
    Rx = R.copy()
    for s in range(S):
        for w in range(W):
            k = ks[s, w]
            rn = oracle.propose_f32((L, L, L), Rx[w, :, k], delta[s, w])[0]
            d1 = _ref_j1(ions, start, fn1, rn.astype(np.float64)) - _ref_j1(ions, start, fn1, Rx[w, :, k].astype(np.float64))
            assert abs(dj[s, w] - dj2only[s, w] - d1) <= 1e-11 * max(1.0, abs(d1)), (s, w)
            if acc[s, w]:
                Rx[w, :, k] = rn
    assert np.array_equal(R2, Rx)
    moved = np.zeros((W, N), bool)
    for s in range(S):
        moved[np.arange(W)[acc[s] == 1], ks[s][acc[s] == 1]] = True
    for w in range(W):
        e = np.nonzero(moved[w])[0]
        o1, _ = oracle.eval_j1(ions, start, R2[w][:, e].T.reshape(-1, 1, 3).astype(np.float64), fn1)
        np.testing.assert_allclose(S1[w][:, e].T, o1[:, 0], rtol=1e-12, atol=1e-12)
        assert np.all(S1[w][:, ~np.pad(moved[w], (0, R.shape[2] - N))] == 0.0)
