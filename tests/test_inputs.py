"""Host-side checks of the seeded input generator (qmcgen) -- no GPU."""
import numpy as np

import qmcgen


def test_positions_in_cell_and_deterministic():
    for dtype in (np.float32, np.float64):
        N = 1000
        L = qmcgen.cell_length(N)
        R = qmcgen.positions(7, [0, 5, 9], N, qmcgen.padded_size(N, 32), L, dtype)
        assert R.dtype == dtype
        assert np.all(R[:, :, :N] >= 0) and np.all(R[:, :, :N] < dtype(L))
        assert np.all(R[:, :, N:] == 0)
        R2 = qmcgen.positions(7, [5], N, qmcgen.padded_size(N, 32), L, dtype)
        assert np.array_equal(R[1], R2[0])          # walker subset independent
        assert not np.array_equal(R[0], R[1])


def test_position_at_matches_positions():
    N, L = 500, qmcgen.cell_length(500)
    R = qmcgen.positions(3, [4], N, 512, L, np.float32)
    i = np.array([0, 17, 499])
    for d in range(3):
        assert np.array_equal(qmcgen.position_at(3, 4, d, i, L, np.float32), R[0, d, i])


def test_cell_is_fp32_exact():
    for N in (14, 1400, 614400, 6144, 4915200):
        L = qmcgen.cell_length(N)
        assert float(np.float32(L)) == L
        assert abs(L ** 3 / N - 1) < 1e-5


def test_uniformity_rough():
    N = 200000
    L = qmcgen.cell_length(N)
    R = qmcgen.positions(1, [0], N, N, L, np.float32)[0] / np.float32(L)
    h, _ = np.histogram(R.ravel(), bins=10, range=(0, 1))
    assert np.all(np.abs(h / h.mean() - 1) < 0.02)


def test_trials_and_k():
    cfg = qmcgen.CONFIGS["C2"]
    R, k, rt, fn = qmcgen.host_instance(cfg, walkers=np.arange(64), P=2, mode="drift")
    assert k.dtype == np.int32 and np.all((k >= 0) & (k < cfg.N))
    assert rt.shape == (64, 2, 3) and rt.dtype == np.float32
    for w in range(64):
        assert np.array_equal(rt[w, 0], R[w, :, k[w]])     # drift mode p=0 is r_k
    assert np.all(rt >= 0) and np.all(rt < np.float32(cfg.L))
    assert fn.coef.shape == (2, 11) and np.all(fn.coef[:, 8:] == 0)
    assert fn.r_cut == cfg.L / 2


def test_config_sizes():
    c3 = qmcgen.CONFIGS["C3"]
    assert c3.W * 3 * c3.Np * 4 == 7549747200           # ~7.55 GB of R
    assert c3.items == 1024 * 614399
    c5 = qmcgen.CONFIGS["C5"]
    assert c5.W * 3 * c5.Np * 4 == 60397977600


def test_oracle_side_generator_matches_qmcgen():
    import oracle
    for dtype in (np.float32, np.float64):
        N, Np = 3001, 3008
        L = qmcgen.cell_length(N)
        a = oracle.gen_positions(9, 40, 5, N, Np, L, dtype, threads=3)
        b = qmcgen.positions(9, np.arange(40, 45), N, Np, L, dtype)
        assert a.dtype == b.dtype and np.array_equal(a, b)


def test_j1_inputs():
    L = qmcgen.cell_length(614400)
    ions, start = qmcgen.make_ions(2, 51200, 51200, L, np.float32)
    assert ions.shape == (3, 51200) and list(start) == [0, 25600, 51200]
    assert np.all(ions >= 0) and np.all(ions < np.float32(L))
    fn1 = qmcgen.make_j1_functor(2, L)
    assert fn1.m == (8, 10) and fn1.r_cut[0] == L / 2 and fn1.r_cut[1] < L / 2
    assert np.all(fn1.coef[0, 8:] == 0) and np.all(fn1.coef[1, 10:] == 0)


def test_spo_table_generators_agree():
    """qmcgen.spo_table (numpy) and the oracle's C twin are bitwise equal; the
    row sampler returns the same rows."""
    import oracle
    a = qmcgen.spo_table(9, 5, 6, 7, 10, 12)
    b = oracle.gen_spo_table(9, 5, 6, 7, 10, 12, threads=3)
    assert np.array_equal(a, b)
    r = qmcgen.spo_table_rows(9, 5, 6, 7, 12, 10, [[4, 5, 6], [0, 0, 0]])
    assert np.array_equal(r[0], a[4, 5, 6]) and np.array_equal(r[1], a[0, 0, 0])
    assert np.all(a[..., 10:] == 0) and a.min() >= -1 and a.max() < 1


def test_sweep_inputs_are_an_ordered_sweep():
    """qmcgen.make_sweep (reading R20): k[s][w] = (k0_w + s) mod N, trial 0 is the
    electron's generated position (no electron moves twice while S <= N), trial 1 is
    inside the cell, u in [0, 1)."""
    N, W, S = 50, 7, 50
    L = qmcgen.cell_length(N)
    Np = qmcgen.padded_size(N, 32)
    R = qmcgen.positions(3, np.arange(W), N, Np, L, np.float32)
    ks, tr, u = qmcgen.make_sweep(3, W, N, L, np.float32, S)
    assert ks.shape == (S, W) and tr.shape == (S, W, 2, 3) and u.shape == (S, W)
    assert np.array_equal(ks, (ks[0][None, :] + np.arange(S)[:, None]) % N)
    for s in range(S):
        assert np.array_equal(tr[s, :, 0, :], R[np.arange(W), :, ks[s]])
    assert np.all((tr[:, :, 1] >= 0) & (tr[:, :, 1] < L))
    assert np.all((u >= 0) & (u < 1)) and u.dtype == np.float64


def test_trial_draws_do_not_depend_on_the_walker_subset():
    """Every make_trials mode gives a walker the same trial points whichever walkers
    are requested (the bench's oracle sample of walkers [0, n) and the GPU run of all
    W must see the same inputs), and make_sweep_moves' streams are independent draws
    of one shape (stream 0 = the default)."""
    N, L = 768, qmcgen.cell_length(768)
    k = qmcgen.make_k(7, 64, N)
    for mode, P in (("move", 1), ("drift", 2), ("noop", 1), ("nlpp", 12)):
        full = qmcgen.make_trials(7, np.arange(64), k, N, L, np.float32, P=P, mode=mode)
        part = qmcgen.make_trials(7, np.arange(10), k[:10], N, L, np.float32, P=P, mode=mode)
        sub = qmcgen.make_trials(7, np.array([3, 40]), k[[3, 40]], N, L, np.float32, P=P, mode=mode)
        assert np.array_equal(full[:10], part), mode
        assert np.array_equal(full[[3, 40]], sub), mode
    a = qmcgen.make_sweep_moves(7, 16, N, 20)
    b = qmcgen.make_sweep_moves(7, 16, N, 20, stream=0)
    c = qmcgen.make_sweep_moves(7, 16, N, 20, stream=1)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    assert np.array_equal(a[0], c[0]) and not np.array_equal(a[1], c[1])     # ordered k, fresh delta
