"""Pins of the NEXT-2 oracle (per-electron 5N J2 state and the accept-side
update, oracle/oracle.c orc_j2_state / orc_accept) against things other than
itself: the numpy+scipy brute-force pair sum (reading R1), finite
differences of it, the from-scratch state after many accepted moves, the
quadratic-functor closed form, and bitwise no-op/reject properties.

PAPER:850 (Alg. 1 L9 "Accept r_k <- r'_k or reject"), PAPER:1305-1306 (R and
Rsoa updated on acceptance), PAPER:1382-1393 (Delta J2, the 5N state).
"""
import numpy as np
import pytest

import oracle
import qmcgen
from test_oracle_pins import ref_j2_total, ref_minimg_27, small_instance


def _moves(seed, W, R, N, L, P_acc=0.7):
    """k, r_new, accept mask for one accept call (harness draws)."""
    rng = np.random.default_rng(seed)
    k = rng.integers(0, N, size=W).astype(np.int32)
    rk = R[np.arange(W), :, k]
    rn = np.mod(rk + rng.normal(0.0, 0.3, size=(W, 3)), L)
    rn = np.where(rn >= L, 0.0, rn)
    acc = (rng.random(W) < P_acc).astype(np.int32)
    return k, rn, acc


@pytest.mark.parametrize("N", [5, 14, 33])
def test_state_sums_to_twice_the_pair_sum(N):
    """sum_e V_e = 2 J2 with J2 = sum_{i<j} U(r_ij) (reading R1) by numpy+scipy."""
    R, _, _, fn = small_instance(N, W=3, seed=60 + N)
    for w in range(3):
        st, _ = oracle.j2_state(R[w], N, N // 2, fn)
        j2 = ref_j2_total(R[w], N, N // 2, fn)
        assert abs(st[0, :N].sum() - 2 * j2) <= 1e-12 * max(1.0, abs(j2))
        assert np.all(st[:, N:] == 0.0)


def test_state_gradient_laplacian_are_derivatives_of_j2():
    """G_e = grad_e J2, L_e = lap_e J2: central differences of the numpy
    brute-force J2 in the position of electron e."""
    N = 20
    R, _, _, fn = small_instance(N, W=1, seed=71)
    R1 = R[0]
    st, ab = oracle.j2_state(R1, N, N // 2, fn)
    h1, h2 = 1e-5 * fn.L[0], 1e-4 * fn.L[0]

    def J(e, shift):
        Rs = R1.copy()
        Rs[:, e] = np.mod(Rs[:, e] + shift, fn.L[0])
        return ref_j2_total(Rs, N, N // 2, fn)

    for e in (0, 7, 13, 19):
        g = np.array([(J(e, h1 * u) - J(e, -h1 * u)) / (2 * h1) for u in np.eye(3)])
        lap = sum((J(e, h2 * u) - 2 * J(e, 0 * u) + J(e, -h2 * u)) / h2 ** 2 for u in np.eye(3))
        assert np.max(np.abs(g - st[1:4, e])) <= 1e-6 * max(ab[1:4, e].max(), 1.0)
        assert abs(lap - st[4, e]) <= 1e-5 * max(ab[4, e], 1.0)


def test_state_of_k_equals_eval_at_r_k():
    """Electron k's state is qj2_eval's (V, G, L) at r_trial = r_k (PAPER:1382,
    Alg. 1 L8): the eval oracle and the state oracle agree."""
    N, W = 30, 4
    R, k, _, fn = small_instance(N, W=W, seed=81)
    rt = R[np.arange(W), :, k].reshape(W, 1, 3)
    out, absout, _ = oracle.eval_j2(R, k, rt, fn, n_total=N, n_up=N // 2)
    for w in range(W):
        st, _ = oracle.j2_state(R[w], N, N // 2, fn)
        err = np.abs(st[:, k[w]] - out[w, 0]) / np.maximum(absout[w, 0], 1.0)
        assert err.max() <= 1e-13


def test_quadratic_functor_closed_form_state():
    """U = r^2 (SURVEY 8(c) pin (iii)): V_e = sum r^2, G_e = 2 sum d (d = r_e - r_j),
    L_e = 6 * (partners inside the cutoff), by 27-image brute force."""
    N = 40
    R, _, _, fn = small_instance(N, W=1, seed=91)
    x = (np.arange(fn.m + 3) - 1) * fn.delta
    fq = qmcgen.Functor(L=fn.L, r_cut=fn.r_cut, m=fn.m, coef=np.stack([x ** 2 - fn.delta ** 2 / 3] * 2))
    st, _ = oracle.j2_state(R[0], N, N // 2, fq)
    pos = R[0, :, :N].T
    for e in range(N):
        j = np.array([i for i in range(N) if i != e])
        r, d = ref_minimg_27(fn.L, pos[j], np.repeat(pos[e:e + 1], j.size, 0))   # d = r_e - r_j
        inside = r < fn.r_cut
        assert abs(st[4, e] - 6 * inside.sum()) <= 1e-10 * max(1, inside.sum())
        np.testing.assert_allclose(st[0, e], (r[inside] ** 2).sum(), rtol=1e-12)
        np.testing.assert_allclose(st[1:4, e], 2 * d[inside].sum(0), atol=1e-10 * N)


@pytest.mark.parametrize("N", [14, 33])
def test_accept_sequence_matches_state_from_scratch(N):
    """50 rounds of batched accept/reject: the incrementally updated state
    equals the state of the final configuration recomputed from scratch, and
    R holds exactly the accepted positions."""
    W = 4
    R, _, _, fn = small_instance(N, W=W, seed=100 + N)
    L = fn.L[0]
    state = np.stack([oracle.j2_state(R[w], N, N // 2, fn)[0] for w in range(W)])
    Rx = R.copy()
    for it in range(50):
        k, rn, acc = _moves(1000 + it, W, Rx, N, L)
        R2, S2, ab = oracle.accept(Rx, state, k, rn, acc, fn, N, N // 2)
        for w in range(W):
            if acc[w]:
                exp = Rx[w].copy()
                exp[:, k[w]] = rn[w]
                assert np.array_equal(R2[w], exp)
            else:
                assert np.array_equal(R2[w], Rx[w]) and np.array_equal(S2[w], state[w])
        Rx, state = R2, S2
    for w in range(W):
        fresh, ab = oracle.j2_state(Rx[w], N, N // 2, fn)
        err = oracle.normalized_error_state(state[w], fresh, ab, fn)
        assert err.max() <= 1e-12


def test_accept_noop_move_is_bitwise_for_partners():
    """r'_k = r_k: every partner's update is T - T = 0 exactly, so their state
    is bitwise unchanged; k's entry becomes the from-scratch value."""
    N, W = 25, 3
    R, _, _, fn = small_instance(N, W=W, seed=121)
    state = np.stack([oracle.j2_state(R[w], N, N // 2, fn)[0] for w in range(W)])
    rng = np.random.default_rng(5)
    state = state + rng.normal(size=state.shape)       # the update is additive: any state works
    k = np.array([0, 12, 24], dtype=np.int32)
    rn = R[np.arange(W), :, k]
    R2, S2, _ = oracle.accept(R, state, k, rn, np.ones(W, np.int32), fn, N, N // 2)
    assert np.array_equal(R2, R)
    for w in range(W):
        others = np.array([i for i in range(state.shape[2]) if i != k[w]])
        assert np.array_equal(S2[w][:, others], state[w][:, others])
        fresh, _ = oracle.j2_state(R[w], N, N // 2, fn)
        np.testing.assert_allclose(S2[w][:, k[w]], fresh[:, k[w]], rtol=1e-13, atol=1e-13)


def test_accept_update_is_the_difference_of_two_evals():
    """For a partner i, the update of V_i is U(|r_i - r'_k|) - U(|r_i - r_k|):
    checked against the scipy functor at 27-image distances."""
    from test_oracle_pins import ref_functor
    N, W = 18, 2
    R, _, _, fn = small_instance(N, W=W, seed=131)
    state = np.zeros((W, 5, R.shape[2]))
    k, rn, _ = _moves(7, W, R, N, fn.L[0])
    _, S2, _ = oracle.accept(R, state, k, rn, np.ones(W, np.int32), fn, N, N // 2)
    for w in range(W):
        for i in range(N):
            if i == k[w]:
                continue
            rn_, _ = ref_minimg_27(fn.L, rn[w:w + 1], R[w, :, i:i + 1].T)
            ro_, _ = ref_minimg_27(fn.L, R[w, :, k[w]:k[w] + 1].T, R[w, :, i:i + 1].T)
            ch = 0 if (i < N // 2) == (k[w] < N // 2) else 1
            dv = ref_functor(fn.coef[ch], fn.m, fn.r_cut, rn_) - ref_functor(fn.coef[ch], fn.m, fn.r_cut, ro_)
            assert abs(S2[w, 0, i] - dv[0]) <= 1e-14 * max(1.0, np.abs(fn.coef).max())
