"""Row padding far beyond the minimum (-m gpu): every entry point addresses
lane i of axis d at d*Np + i, so an Np much larger than N (here up to 3N + 4096)
must change nothing -- and the padding lanes, filled with NaN, must never be read
as sources (one NaN term would poison a whole sum) nor written."""
import os

import numpy as np
import pytest
import torch

import oracle
import qmcgen
from sweep_check import check_sweep

pytestmark = pytest.mark.gpu

TOL = {np.float32: 1e-5, np.float64: 1e-12}
THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def q():
    import paper_1708_02645_b200 as q
    q.device_check()
    return q


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def padded(N, W, seed, dtype, extra):
    L = qmcgen.cell_length(N)
    vw = 4 if dtype == np.float32 else 2
    Np = qmcgen.padded_size(N, vw) + extra
    R = qmcgen.positions(seed, np.arange(W), N, Np, L, dtype)
    R[:, :, N:] = np.nan
    return R, L, Np


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("N,W", [(700, 64), (9000, 5), (250000, 2)])
def test_eval_wide_padding(q, dtype, N, W):
    for extra in (4096, 2 * N + 4096):
        R, L, Np = padded(N, W, 40 + N, dtype, extra)
        k = qmcgen.make_k(40 + N, W, N)
        rt = qmcgen.make_trials(40 + N, np.arange(W), k, N, L, dtype, P=2, mode="drift")
        fn = qmcgen.make_functor(40 + N, L)
        out = q.eval(dev(R), dev(k), dev(rt), fn, N, N // 2).cpu().numpy()
        assert np.all(np.isfinite(out))
        orc, absout, _ = oracle.eval_j2(R, k, rt, fn, N, N // 2, threads=THREADS)
        assert oracle.normalized_error(out, orc, absout, fn).max() <= TOL[dtype]


def test_accept_wide_padding(q):
    N, W, dtype = 3000, 12, np.float32
    R, L, Np = padded(N, W, 50, dtype, 2 * N + 4096)
    k = qmcgen.make_k(50, W, N)
    rt = qmcgen.make_trials(50, np.arange(W), k, N, L, dtype)
    fn = qmcgen.make_functor(50, L)
    rng = np.random.default_rng(51)
    state = rng.normal(size=(W, 5, Np)).astype(dtype)
    state[:, :, N:] = np.nan
    acc = (np.arange(W) % 2).astype(np.int32)
    Rd, Sd = dev(R), dev(state)
    out = q.eval(Rd, dev(k), dev(rt), fn, N, N // 2)
    q.accept(Rd, Sd, dev(k), dev(rt), dev(acc), out, fn, N, N // 2)
    Rg, Sg = Rd.cpu().numpy(), Sd.cpu().numpy()
    assert np.all(np.isnan(Rg[:, :, N:])) and np.all(np.isnan(Sg[:, :, N:]))      # padding untouched
    R2, S2, ab = oracle.accept(R[:, :, :N].copy(), state[:, :, :N].copy(), k, rt[:, 0], acc, fn, N, N // 2)
    assert np.array_equal(Rg[:, :, :N].astype(np.float64), R2)
    a = acc != 0
    assert oracle.normalized_error_state(Sg[a][:, :, :N], S2[a], ab[a], fn).max() <= 1e-5


def test_state_init_and_sweep_wide_padding(q):
    N, W = 500, 4
    R, L, Np = padded(N, W, 60, np.float32, 2 * N + 4096)
    fn = qmcgen.make_functor(60, L)
    Sd = torch.full((W, 5, Np), float("nan"), dtype=torch.float32, device="cuda")
    q.state_init(dev(R), Sd, fn, N, N // 2)
    Sg = Sd.cpu().numpy()
    assert np.all(np.isnan(Sg[:, :, N:])) and np.all(np.isfinite(Sg[:, :, :N]))
    for w in range(W):
        st, ab = oracle.j2_state(R[w][:, :N].astype(np.float64), N, N // 2, fn)
        assert oracle.normalized_error_state(Sg[w][:, :N], st, ab, fn).max() <= 1e-5
    ks, delta, u = qmcgen.make_sweep_moves(61, W, N, 2 * N, order="random")
    # the sweep oracle's rows are the first N lanes; the GPU side keeps the NaN padding
    check_sweep(q, np.nan_to_num(R, nan=0.0), np.nan_to_num(Sg, nan=0.0), ks, delta, u, fn, N, N // 2)
    Rd, Sd2 = dev(R), dev(Sg)
    q.sweep(Rd, Sd2, dev(ks), dev(delta), dev(u), fn, N, N // 2)
    assert np.all(np.isnan(Rd.cpu().numpy()[:, :, N:])) and np.all(np.isnan(Sd2.cpu().numpy()[:, :, N:]))
    assert np.all(np.isfinite(Rd.cpu().numpy()[:, :, :N])) and np.all(np.isfinite(Sd2.cpu().numpy()[:, :, :N]))


def test_j1_wide_ion_padding(q):
    """The ion rows [3][Np_ion] with Np_ion far beyond n_ions (NaN padding)."""
    for n_ions in (64, 9000):
        N = 768
        L = qmcgen.cell_length(N)
        Np_ion = qmcgen.padded_size(n_ions, 4) + 3 * n_ions + 4096
        ions, start = qmcgen.make_ions(70 + n_ions, n_ions, Np_ion, L, np.float32, n_species=2)
        ions[:, n_ions:] = np.nan
        fn1 = qmcgen.make_j1_functor(70 + n_ions, L, n_species=2)
        k = qmcgen.make_k(71, 64, N)
        rt = qmcgen.make_trials(71, np.arange(64), k, N, L, np.float32)
        out = q.eval_j1(dev(ions), start, dev(rt), fn1).cpu().numpy()
        assert np.all(np.isfinite(out))
        orc, absout = oracle.eval_j1(ions[:, :n_ions].astype(np.float64), start, rt.astype(np.float64), fn1)
        assert oracle.normalized_error_j1(out, orc, absout, fn1).max() <= 1e-5


@pytest.mark.parametrize("N,W", [(250000, 2), (6144, 4096)])
def test_eval_and_accept_16_byte_aligned_rows(q, N, W):
    """Rows that start 16- but not 32-byte aligned take the 128-bit path of the
    kernels that otherwise read 256 bits at a time (CTA kernel, compact warp
    kernel, accept kernel): the same results as the oracle."""
    L = qmcgen.cell_length(N)
    Np = qmcgen.padded_size(N, 8)
    R = qmcgen.positions(80 + N, np.arange(W), N, Np, L, np.float32)
    k = qmcgen.make_k(80 + N, W, N)
    rt = qmcgen.make_trials(80 + N, np.arange(W), k, N, L, np.float32)
    fn = qmcgen.make_functor(80 + N, L)
    big = torch.empty(R.size + 4, dtype=torch.float32, device="cuda")
    Rd = big[4:].view(W, 3, Np)                       # 16 bytes past a 256-byte boundary
    assert Rd.data_ptr() % 32 == 16
    Rd.copy_(dev(R))
    out = q.eval(Rd, dev(k), dev(rt), fn, N, N // 2).cpu().numpy()
    sample = np.r_[0:2, W - 2:W] if W > 16 else np.arange(W)
    orc, absout, _ = oracle.eval_j2(R[sample], k[sample], rt[sample], fn, N, N // 2, threads=THREADS)
    assert oracle.normalized_error(out[sample], orc, absout, fn).max() <= 1e-5
    if W <= 16:
        rng = np.random.default_rng(81)
        state = rng.normal(size=(W, 5, Np)).astype(np.float32)
        bigs = torch.empty(state.size + 4, dtype=torch.float32, device="cuda")
        Sd = bigs[4:].view(W, 5, Np)
        Sd.copy_(dev(state))
        acc = np.ones(W, np.int32)
        q.accept(Rd, Sd, dev(k), dev(rt), dev(acc), q.eval(Rd, dev(k), dev(rt), fn, N, N // 2), fn, N, N // 2)
        R2, S2, ab = oracle.accept(R, state, k, rt[:, 0], acc, fn, N, N // 2)
        assert np.array_equal(Rd.cpu().numpy().astype(np.float64), R2)
        assert oracle.normalized_error_state(Sd.cpu().numpy()[:, :, :N], S2[:, :, :N], ab[:, :, :N], fn).max() <= 1e-5
