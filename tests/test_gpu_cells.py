"""Orthorhombic (non-cubic) cells through every J2 entry point (-m gpu).

The configurations all use cubic cells, so an axis mix-up (one axis's L or
half-width used for another) would pass them unnoticed; here L = (3, 4.5, 6.25)
(and a permutation of it), positions uniform in each axis's own [0, L_d),
against the oracle, which takes the cell per axis."""
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
CELLS = [(3.0, 4.5, 6.25), (6.25, 3.0, 4.5)]


@pytest.fixture(scope="module")
def q():
    import paper_1708_02645_b200 as q
    q.device_check()
    return q


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def cell_points(seed, W, n, n_pad, L, dtype):
    """[W][3][n_pad] points uniform in [0, L_d) per axis (harness draw; padding 0)."""
    u = qmcgen.positions(seed, np.arange(W), n, n_pad, 1.0, np.float64)
    out = np.zeros((W, 3, n_pad), dtype=dtype)
    for d in range(3):
        x = (u[:, d, :n] * L[d]).astype(dtype)
        below = np.nextafter(dtype(L[d]), dtype(0))
        out[:, d, :n] = np.minimum(x, below)
    return out


def functor(seed, L, m=8):
    fn = qmcgen.make_functor(seed, min(L), m)
    return qmcgen.Functor(L=tuple(float(x) for x in L), r_cut=min(L) / 2.0, m=m, coef=fn.coef)


@pytest.mark.parametrize("L", CELLS)
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("N,W", [(300, 64), (30000, 3), (250000, 2)])
def test_eval_orthorhombic(q, L, dtype, N, W):
    vw = 4 if dtype == np.float32 else 2
    Np = qmcgen.padded_size(N, vw)
    R = cell_points(11 + N, W, N, Np, L, dtype)
    k = qmcgen.make_k(11 + N, W, N)
    rt = cell_points(12 + N, W, 2, 2, L, dtype).transpose(0, 2, 1).copy()     # two trials per walker
    fn = functor(13 + N, L)
    out = q.eval(dev(R), dev(k), dev(rt), fn, N, N // 2).cpu().numpy()
    orc, absout, _ = oracle.eval_j2(R, k, rt, fn, N, N // 2, threads=THREADS)
    assert oracle.normalized_error(out, orc, absout, fn).max() <= TOL[dtype]


@pytest.mark.parametrize("L", CELLS)
def test_accept_orthorhombic(q, L):
    N, W = 5000, 16
    dtype = np.float32
    Np = qmcgen.padded_size(N, 4)
    R = cell_points(21, W, N, Np, L, dtype)
    k = qmcgen.make_k(21, W, N)
    rt = cell_points(22, W, 1, 1, L, dtype).transpose(0, 2, 1).copy()
    fn = functor(23, L)
    rng = np.random.default_rng(24)
    state = rng.normal(size=(W, 5, Np)).astype(dtype)
    acc = (np.arange(W) % 3 != 0).astype(np.int32)
    Rd, Sd = dev(R), dev(state)
    out = q.eval(Rd, dev(k), dev(rt), fn, N, N // 2)
    q.accept(Rd, Sd, dev(k), dev(rt), dev(acc), out, fn, N, N // 2)
    R2, S2, ab = oracle.accept(R, state, k, rt[:, 0], acc, fn, N, N // 2)
    assert np.array_equal(Rd.cpu().numpy().astype(np.float64), R2)
    a = acc != 0
    err = oracle.normalized_error_state(Sd.cpu().numpy()[a][:, :, :N], S2[a][:, :, :N], ab[a][:, :, :N], fn)
    assert err.max() <= TOL[dtype]


@pytest.mark.parametrize("L", CELLS)
def test_state_init_and_sweep_orthorhombic(q, L):
    """qj2_state_init and two random-order sweeps (the proposal wraps each axis in
    its own L_d) against the oracle."""
    N, W = 600, 6
    Np = qmcgen.padded_size(N, 32)
    R = cell_points(31, W, N, Np, L, np.float32)
    fn = functor(32, L)
    Sd = torch.zeros((W, 5, Np), dtype=torch.float32, device="cuda")
    q.state_init(dev(R), Sd, fn, N, N // 2)
    Sg = Sd.cpu().numpy()
    for w in range(W):
        st, ab = oracle.j2_state(R[w].astype(np.float64), N, N // 2, fn)
        assert oracle.normalized_error_state(Sg[w][:, :N], st[:, :N], ab[:, :N], fn).max() <= 1e-5
    ks, delta, u = qmcgen.make_sweep_moves(33, W, N, 2 * N, order="random", sigma=0.3)
    check_sweep(q, R, Sg, ks, delta, u, fn, N, N // 2)
