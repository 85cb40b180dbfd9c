"""NEXT-1 GPU parity: one-body Jastrow over the electron-ion (AB) row
(qj2_eval_j1) vs the CPU oracle (oracle.eval_j1), element by element, same
tolerance as J2 (normalized by the absolute-term sums; 1e-5 fp32, 1e-12 fp64)."""
import numpy as np
import pytest
import torch

import oracle
import qmcgen

pytestmark = pytest.mark.gpu
TOL = {np.float32: 1e-5, np.float64: 1e-12}


@pytest.fixture(scope="module")
def q():
    import paper_1708_02645_b200 as q
    q.device_check()
    return q


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def j1_case(n_ions, W, seed, dtype, S=2, P=1, mode="move", m=(8, 10, 6, 12), rcut=(0.5, 0.4, 0.3, 0.45)):
    N = max(12 * n_ions, 64)
    L = qmcgen.cell_length(N)
    vw = 4 if dtype == np.float32 else 2
    ions, start = qmcgen.make_ions(seed, n_ions, qmcgen.padded_size(n_ions, vw), L, dtype, n_species=S)
    fn1 = qmcgen.make_j1_functor(seed, L, n_species=S, m=m, rcut_frac=rcut)
    k = qmcgen.make_k(seed, W, N)
    rt = qmcgen.make_trials(seed, np.arange(W), k, N, L, dtype, P=P, mode=mode)
    return ions, start, rt, fn1


def check(q, ions, start, rt, fn1, dtype, sample=None, **kw):
    res = q.eval_j1(dev(ions), start, dev(rt), fn1, **kw)
    out = (res[0] if isinstance(res, tuple) else res).cpu().numpy()
    w = np.arange(rt.shape[0]) if sample is None else np.asarray(sample)
    orc, absout = oracle.eval_j1(ions.astype(np.float64), start, rt[w].astype(np.float64), fn1)
    err = oracle.normalized_error_j1(out[w], orc, absout, fn1)
    assert np.all(np.isfinite(out))
    assert err.max() <= TOL[dtype], f"max normalized error {err.max():.3e}"
    return res, orc


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n_ions", [1, 5, 32, 1000, 8193, 51200])
def test_j1_sizes(q, dtype, n_ions):
    ions, start, rt, fn1 = j1_case(n_ions, 9, seed=500 + n_ions, dtype=dtype)
    check(q, ions, start, rt, fn1, dtype)


@pytest.mark.parametrize("m", [17, 36, 64])
def test_j1_fine_species_functors_fp32(q, m):
    """An fp32 species functor finer than m = 16 takes the fp64 geometry in the
    small-ion kernel: the 1e-5 bar holds where one or two ions
    make the whole sum."""
    for n_ions, S in ((1, 1), (2, 2), (5, 3), (64, 2)):
        ions, start, rt, fn1 = j1_case(n_ions, 2048, seed=700 + m + n_ions, dtype=np.float32, S=S,
                                       m=(m, 8, m, 12))
        check(q, ions, start, rt, fn1, np.float32)


@pytest.mark.parametrize("S", [1, 3, 4])
def test_j1_species_counts_and_straddling(q, S):
    # species boundaries at n*s//S land inside sub-tiles (masked multi-species path)
    for dtype in (np.float32, np.float64):
        ions, start, rt, fn1 = j1_case(20011, 5, seed=600 + S, dtype=dtype, S=S)
        check(q, ions, start, rt, fn1, dtype)


def test_j1_warp_mapping_many_walkers(q):
    for dtype in (np.float32, np.float64):
        ions, start, rt, fn1 = j1_case(640, 4096, seed=7, dtype=dtype)
        check(q, ions, start, rt, fn1, dtype, sample=np.arange(0, 4096, 97))


@pytest.mark.parametrize("P", [2, 3])
def test_j1_multi_trial_and_ratio(q, P):
    ions, start, rt, fn1 = j1_case(3000, 11, seed=800 + P, dtype=np.float64, P=P, mode="drift")
    res, orc = check(q, ions, start, rt, fn1, np.float64, ratio=True)
    out, rat = res
    rat = rat.cpu().numpy()
    assert np.all(rat[:, 0, 0] == 0.0)
    dj = orc[:, 1, 0] - orc[:, 0, 0]                     # Delta J1
    assert np.max(np.abs(rat[:, 1, 0] - dj)) < 1e-12 * max(1.0, np.abs(orc[:, :, 0]).max())


def test_j1_ab_row_output(q):
    ions, start, rt, fn1 = j1_case(3001, 4, seed=9, dtype=np.float32)
    res, _ = check(q, ions, start, rt, fn1, np.float32, row=True)
    row = res[1].cpu().numpy()
    L = fn1.L[0]
    n = int(start[-1])
    for w in range(4):
        o = oracle.min_image(fn1.L, np.repeat(rt[w, :1].astype(np.float64), n, 0), ions[:, :n].T.astype(np.float64))
        tie = np.abs(np.abs(o[:, 1:]) - L / 2) <= 4 * np.spacing(np.float32(L))
        assert np.all((row[w, 0, 1:, :n].T == o[:, 1:].astype(np.float32)) | tie)
        assert np.all(np.abs(row[w, 0, 0, :n] - o[:, 0].astype(np.float32)) <= 3 * np.spacing(o[:, 0].astype(np.float32)))


def test_j1_validation(q):
    ions, start, rt, fn1 = j1_case(100, 3, seed=1, dtype=np.float32)
    with pytest.raises(q.QJ2Error):
        q.eval_j1(dev(ions), [0, 60, 50], dev(rt), fn1)          # not nondecreasing
    with pytest.raises(q.QJ2Error):
        q.eval_j1(dev(ions), [1, 50, 100], dev(rt), fn1)         # must start at 0


# ---------------------------------------------------------------------------
# Small ion sets: the thread-per-(walker, trial) kernel (ions in shared memory)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n_ions,S", [(64, 2), (33, 3), (1500, 2), (4096, 4)])
def test_j1_thread_kernel_many_walkers(q, dtype, n_ions, S):
    """NiO-64-sized ion sets (64 ions, Ni and O), a set whose staged ions plus
    the static functor table just pass the 48 KB default (1500 fp64 ions), and
    the largest staged set, many walkers; sampled walkers vs the oracle."""
    ions, start, rt, fn1 = j1_case(n_ions, 20000, seed=900 + n_ions, dtype=dtype, S=S)
    check(q, ions, start, rt, fn1, dtype, sample=np.r_[0:40, 19990:20000])


def test_j1_thread_kernel_nlpp_and_ratio(q):
    """P = 12 quadrature points per walker through the thread kernel; ratios
    against V_cur and against trial 0 (second launch)."""
    import qmcgen as g
    ions, start, _, fn1 = j1_case(64, 300, seed=31, dtype=np.float32)
    N = 768
    k = g.make_k(31, 300, N)
    rt = g.make_trials(31, np.arange(300), k, N, g.cell_length(N), np.float32, P=12, mode="nlpp")
    rt = np.mod(rt, np.float32(fn1.L[0])).astype(np.float32)
    res, orc = check(q, ions, start, rt, fn1, np.float32)
    vcur = dev(orc[:, 0, 0].copy())
    _, r1 = q.eval_j1(dev(ions), start, dev(rt), fn1, V_cur=vcur, ratio=True)
    _, r0 = q.eval_j1(dev(ions), start, dev(rt), fn1, ratio=True)
    out = res.cpu().numpy()
    np.testing.assert_allclose(r1.cpu().numpy()[:, :, 0], out[:, :, 0] - orc[:, :1, 0], atol=1e-9)
    assert np.all(r0.cpu().numpy()[:, 0, 0] == 0.0)


def test_j1_thread_and_warp_kernels_agree(q):
    """The thread-per-trial kernel (small ion sets) and the shared warp kernel (taken
    with row output, or for > 4096 ions) agree."""
    ions, start, rt, fn1 = j1_case(64, 5000, seed=41, dtype=np.float32)
    a = q.eval_j1(dev(ions), start, dev(rt), fn1).cpu().numpy()
    b = q.eval_j1(dev(ions), start, dev(rt), fn1, row=True)[0].cpu().numpy()
    orc, absout = oracle.eval_j1(ions.astype(np.float64), start, rt[:50].astype(np.float64), fn1)
    assert oracle.normalized_error_j1(a[:50], orc, absout, fn1).max() <= 1e-5
    assert oracle.normalized_error_j1(b[:50], orc, absout, fn1).max() <= 1e-5
    assert np.max(np.abs(a - b)) <= 1e-4 * np.abs(a).max()


def test_j1_sweep_batch_full_size_every_point(q):
    """The J1S bench workload at full size (786,432 trial points x 64 ions,
    fp32) in the bench launch configuration; every trial point vs the oracle."""
    import qmcgen as g
    cfg = g.J1_CONFIGS["J1S"]
    ions, start = g.make_ions(cfg.seed, cfg.n_ions, g.padded_size(cfg.n_ions, 4), cfg.L, np.float32,
                              n_species=cfg.n_species)
    fn1 = g.make_j1_functor(cfg.seed, cfg.L, n_species=cfg.n_species)
    ids = np.arange(cfg.W)
    rt = g.make_trials(cfg.seed, ids, (ids % cfg.N).astype(np.int32), cfg.N, cfg.L, np.float32)
    check(q, ions, start, rt, fn1, np.float32)
