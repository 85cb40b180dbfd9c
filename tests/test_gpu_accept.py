"""GPU parity of NEXT-2 (accept-side update of R and the 5N J2 state,
qj2_accept; Metropolis decision, qj2_metropolis) against the CPU oracle
(oracle.accept / oracle.j2_state), through the C ABI (-m gpu; needs a B200).

Tolerance: per state entry |s_gpu - s_orc| / max(A, F) <= 1e-5 (fp32 state)
or 1e-12 (fp64), A = |s_old| + |T(r')| + |T(r)| (the oracle's bound), F the
functor scale.  Positions: bit-exact.  Rejected walkers and padding slots:
bitwise untouched.
"""
import os

import numpy as np
import pytest
import torch

import oracle
import qmcgen

pytestmark = pytest.mark.gpu

TOL = {np.float32: 1e-5, np.float64: 1e-12}
THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def q():
    import paper_1708_02645_b200 as q
    assert torch.cuda.is_available()
    q.device_check()
    return q


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def setup(N, W, seed, dtype, n_up=None, pad_fill=7.0, m=8):
    L = qmcgen.cell_length(N)
    vw = 4 if dtype == np.float32 else 2
    Np = qmcgen.padded_size(N, vw)
    R = qmcgen.positions(seed, np.arange(W), N, Np, L, dtype)
    k = qmcgen.make_k(seed, W, N)
    rt = qmcgen.make_trials(seed, np.arange(W), k, N, L, dtype)
    fn = qmcgen.make_functor(seed, L, m)
    rng = np.random.default_rng(seed)
    state = rng.normal(size=(W, 5, Np)).astype(dtype)        # the update is additive: any state works
    state[:, :, N:] = pad_fill
    acc = (rng.random(W) < 0.75).astype(np.int32)
    return R, k, rt, fn, state, acc, (N // 2 if n_up is None else n_up)


def run_gpu(q, R, k, rt, fn, state, acc, N, n_up, **kw):
    Rd, Sd = dev(R), dev(state)
    out = q.eval(Rd, dev(k), dev(rt), fn, N, n_up)
    q.accept(Rd, Sd, dev(k), dev(rt), dev(acc), out, fn, N, n_up, **kw)
    torch.cuda.synchronize()
    return Rd.cpu().numpy(), Sd.cpu().numpy(), out.cpu().numpy()


def compare(R, state, acc, N, fn, dtype, Rg, Sg, R2, S2, ab):
    assert np.array_equal(Rg.astype(np.float64), R2), "positions must be bit-exact"
    rej = acc == 0
    assert np.array_equal(Sg[rej], state[rej]), "rejected walkers must be untouched"
    assert np.array_equal(Sg[:, :, N:], state[:, :, N:]), "padding must be untouched"
    a = ~rej
    if not a.any():
        return
    err = oracle.normalized_error_state(Sg[a][:, :, :N], S2[a][:, :, :N], ab[a][:, :, :N], fn)
    assert np.all(np.isfinite(Sg[a][:, :, :N]))
    assert err.max() <= TOL[dtype], f"max normalized error {err.max():.3e}"


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("N", [2, 3, 14, 17, 1400, 4095, 8192, 8193, 20001])
def test_accept_parity(q, dtype, N):
    W = 33
    R, k, rt, fn, state, acc, n_up = setup(N, W, 400 + N, dtype)
    Rg, Sg, _ = run_gpu(q, R, k, rt, fn, state, acc, N, n_up)
    R2, S2, ab = oracle.accept(R, state, k, rt[:, 0], acc, fn, N, n_up)
    compare(R, state, acc, N, fn, dtype, Rg, Sg, R2, S2, ab)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("m", [4, 13, 64])
def test_accept_functor_resolution(q, dtype, m):
    """Per-entry parity for fine functor grids (t = r/delta up to m = 64): the
    accept path forms r and t in fp64."""
    R, k, rt, fn, state, acc, n_up = setup(1400, 64, 700 + m, dtype, m=m)
    Rg, Sg, _ = run_gpu(q, R, k, rt, fn, state, acc, 1400, n_up)
    R2, S2, ab = oracle.accept(R, state, k, rt[:, 0], acc, fn, 1400, n_up)
    compare(R, state, acc, 1400, fn, dtype, Rg, Sg, R2, S2, ab)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_accept_k_at_tile_and_spin_boundaries(q, dtype):
    N = 3 * 8192 + 5
    ks = np.array([0, 1, 4095, 4096, 8191, 8192, 8193, 16384, N // 2 - 1, N // 2, N - 1], np.int32)
    W = ks.size
    R, _, _, fn, state, _, _ = setup(N, W, 17, dtype)
    L = qmcgen.cell_length(N)
    rt = qmcgen.make_trials(17, np.arange(W), ks, N, L, dtype)
    acc = np.ones(W, np.int32)
    for n_up in (N // 2, 8192, 0, N):
        Rg, Sg, _ = run_gpu(q, R, ks, rt, fn, state, acc, N, n_up)
        R2, S2, ab = oracle.accept(R, state, ks, rt[:, 0], acc, fn, N, n_up)
        compare(R, state, acc, N, fn, dtype, Rg, Sg, R2, S2, ab)


def test_accept_with_caller_r_old_and_empty(q):
    N, W, dtype = 5000, 12, np.float32
    R, k, rt, fn, state, acc, n_up = setup(N, W, 23, dtype)
    r_old = np.ascontiguousarray(R[np.arange(W), :, k])
    Rg, Sg, _ = run_gpu(q, R, k, rt, fn, state, acc, N, n_up, r_old=dev(r_old))
    R2, S2, ab = oracle.accept(R, state, k, rt[:, 0], acc, fn, N, n_up)
    compare(R, state, acc, N, fn, dtype, Rg, Sg, R2, S2, ab)
    # W = 0 is a no-op
    e = torch.zeros((0, 3, 16), dtype=torch.float32, device="cuda")
    q.accept(e, torch.zeros((0, 5, 16), dtype=torch.float32, device="cuda"),
             torch.zeros(0, dtype=torch.int32, device="cuda"), torch.zeros((0, 3), device="cuda"),
             torch.zeros(0, dtype=torch.int32, device="cuda"), torch.zeros((0, 5), dtype=torch.float64,
                                                                           device="cuda"), fn, 16, 8)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_accept_sharded_slices(q, dtype):
    """Per-rank calls of a source-axis split: every slice updates its partners;
    only the slice holding k commits r'_k and state_k (r_old from the caller)."""
    N, W = 30000, 16
    R, k, rt, fn, state, acc, n_up = setup(N, W, 29, dtype)
    out = q.eval(dev(R), dev(k), dev(rt), fn, N, n_up)          # V, G, L at r'_k over all sources
    r_old = dev(np.ascontiguousarray(R[np.arange(W), :, k]))
    R2, S2, ab = oracle.accept(R, state, k, rt[:, 0], acc, fn, N, n_up)
    vw = 4 if dtype == np.float32 else 2
    for G in (2, 3):
        bounds = [N * g // G for g in range(G + 1)]
        Rg = np.zeros_like(R)
        Sg = np.zeros_like(state)
        for a, b in zip(bounds[:-1], bounds[1:]):
            Np = qmcgen.padded_size(b - a, vw)
            Rs = np.zeros((W, 3, Np), dtype)
            Rs[:, :, :b - a] = R[:, :, a:b]
            Ss = np.zeros((W, 5, Np), dtype)
            Ss[:, :, :b - a] = state[:, :, a:b]
            Rd, Sd = dev(Rs), dev(Ss)
            q.accept(Rd, Sd, dev(k), dev(rt), dev(acc), out, fn, N, n_up, i_offset=a, n_local=b - a, r_old=r_old)
            Rg[:, :, a:b] = Rd.cpu().numpy()[:, :, :b - a]
            Sg[:, :, a:b] = Sd.cpu().numpy()[:, :, :b - a]
        Rg[:, :, N:] = R[:, :, N:]
        Sg[:, :, N:] = state[:, :, N:]
        compare(R, state, acc, N, fn, dtype, Rg, Sg, R2, S2, ab)


def test_metropolis_decisions(q):
    """accept = u < rho^2 (Alg. 1 L9, symmetric proposal, J2-only Psi): equal
    to the oracle-side decision wherever u is not within 1e-9 of rho^2."""
    N, W = 3000, 4096
    R, k, rt, fn, _, _, n_up = setup(N, 256, 31, np.float64)
    k = qmcgen.make_k(31, W, N)
    R = qmcgen.positions(31, np.arange(W), N, R.shape[2], fn.L[0], np.float64)
    rt = qmcgen.make_trials(31, np.arange(W), k, N, fn.L[0], np.float64, P=2, mode="drift")
    u = np.random.default_rng(3).random(W)
    out, ratio = q.eval(dev(R), dev(k), dev(rt), fn, N, n_up, ratio=True)
    # ratio of trial 1 relative to trial 0 (V(r'_k) - V(r_k))
    acc = q.metropolis(ratio, dev(u), trial=1).cpu().numpy()
    orc, _, _ = oracle.eval_j2(R, k, rt, fn, N, n_up, threads=THREADS)
    rho2 = np.exp(orc[:, 1, 0] - orc[:, 0, 0]) ** 2
    clear = np.abs(u - rho2) > 1e-9 * np.maximum(rho2, 1e-300)
    assert clear.mean() > 0.99
    assert np.array_equal(acc[clear], (u < rho2)[clear].astype(np.int32))
    assert 0 < acc.sum() < W


def test_sweep_matches_state_from_scratch(q):
    """20 rounds of eval -> metropolis -> accept on the GPU (fp64, N = 64),
    started from the oracle's from-scratch state: the decisions equal the
    oracle's own, the final state equals the from-scratch state of the final
    configuration, and R is the oracle's sequence of accepted moves."""
    N, W, dtype = 64, 8, np.float64
    L = qmcgen.cell_length(N)
    Np = qmcgen.padded_size(N, 2)
    R = qmcgen.positions(41, np.arange(W), N, Np, L, dtype)
    fn = qmcgen.make_functor(41, L)
    state = np.stack([oracle.j2_state(R[w], N, N // 2, fn)[0] for w in range(W)])
    Rd, Sd = dev(R), dev(state)
    Rh, Sh = R.copy(), state.copy()
    for it in range(20):
        k = qmcgen.make_k(1000 + it, W, N)
        rng = np.random.default_rng(2000 + it)
        rk = Rh[np.arange(W), :, k]
        rn = np.mod(rk + rng.normal(0, 0.4, size=(W, 3)), L)
        rn = np.where(rn >= L, 0.0, rn)[:, None, :]
        u = rng.random(W)
        out, ratio = q.eval(Rd, dev(k), dev(rn), fn, N, N // 2, V_cur=Sd[torch.arange(W), 0, dev(k).long()].contiguous(),
                            ratio=True)
        acc = q.metropolis(ratio, dev(u))
        q.accept(Rd, Sd, dev(k), dev(rn), acc, out, fn, N, N // 2)
        # the oracle side takes its own decision from its own values
        orc, _, _ = oracle.eval_j2(Rh, k, rn, fn, N, N // 2)
        rho2 = np.exp(orc[:, 0, 0] - Sh[np.arange(W), 0, k]) ** 2
        a = (u < rho2).astype(np.int32)
        clear = np.abs(u - rho2) > 1e-9 * rho2
        assert np.array_equal(acc.cpu().numpy()[clear], a[clear])
        Rh, Sh, _ = oracle.accept(Rh, Sh, k, rn[:, 0], a, fn, N, N // 2)
    torch.cuda.synchronize()
    assert np.array_equal(Rd.cpu().numpy(), Rh)
    Sg = Sd.cpu().numpy()
    for w in range(W):
        fresh, ab = oracle.j2_state(Rh[w], N, N // 2, fn)
        assert oracle.normalized_error_state(Sg[w][:, :N], fresh[:, :N], ab[:, :N], fn).max() <= 1e-11


def test_accept_C3_full_size_sampled(q):
    """The bench's sweep step at full C3 size (N = 614,400, W = 1024, fp32):
    eval -> accept (every 7th walker rejected), zero initial state; 96 walkers
    (both ends, the middle) checked in full against the oracle (which
    regenerates their positions with its own C generator)."""
    cfg = qmcgen.CONFIGS["C3"]
    R = q.gen_positions(cfg.seed, cfg.W, cfg.N, cfg.Np, cfg.L, torch.float32)
    k = qmcgen.make_k(cfg.seed, cfg.W, cfg.N)
    rt = qmcgen.make_trials(cfg.seed, np.arange(cfg.W), k, cfg.N, cfg.L, np.float32)
    fn = qmcgen.make_functor(cfg.seed, cfg.L, cfg.m)
    S = torch.zeros((cfg.W, 5, cfg.Np), dtype=torch.float32, device="cuda")
    acc = np.ones(cfg.W, np.int32)
    acc[1::7] = 0
    out = q.eval(R, dev(k), dev(rt), fn, cfg.N, cfg.n_up)
    q.accept(R, S, dev(k), dev(rt), dev(acc), out, fn, cfg.N, cfg.n_up)
    torch.cuda.synchronize()
    for w0 in list(range(0, 32, 8)) + list(range(480, 544, 16)) + [992, 1000, 1008, 1016]:   # 96 walkers
        n = 8
        Rw = oracle.gen_positions(cfg.seed, w0, n, cfg.N, cfg.Np, cfg.L, np.float32, threads=THREADS)
        Sw = np.zeros((n, 5, cfg.Np), np.float32)
        sl = slice(w0, w0 + n)
        R2, S2, ab = oracle.accept(Rw, Sw, k[sl], rt[sl, 0], acc[sl], fn, cfg.N, cfg.n_up)
        compare(Rw, Sw, acc[sl], cfg.N, fn, np.float32, R[sl].cpu().numpy(), S[sl].cpu().numpy(), R2, S2, ab)
    del R, S
    torch.cuda.empty_cache()


def test_sweep_captured_as_cuda_graph_equals_eager(q):
    """A full particle-by-particle sweep (N moves: eval P = 2 -> Metropolis ->
    accept) captured once in a CUDA graph and replayed gives bitwise the same
    positions, state and decisions as the same calls launched eagerly (the
    bench's N64S path)."""
    N, W = 96, 64
    L = qmcgen.cell_length(N)
    Np = qmcgen.padded_size(N, 32)
    fn = q.Functor.of(qmcgen.make_functor(3, L))
    ks, tr, u = qmcgen.make_sweep(3, W, N, L, np.float32, N)
    ks, tr, u = dev(ks), dev(tr), dev(u)
    R0 = dev(qmcgen.positions(3, np.arange(W), N, Np, L, np.float32))
    ws = q.Workspace(q.workspace_size(W, 2, N, torch.float32))
    wsa = q.Workspace(1 << 16)

    def run(R, S, out, ratio, acc, accs):
        for s in range(N):
            if s % 2:      # both move forms: separate ratio/Metropolis/accept launches and the fused one
                q.eval(R, ks[s], tr[s], fn, N, N // 2, ratio=True, out=out, ratio_out=ratio, workspace=ws)
                q.metropolis(ratio, u[s], acc, trial=1)
                q.accept(R, S, ks[s], tr[s], acc, out, fn, N, N // 2, trial=1, workspace=wsa)
            else:
                q.eval(R, ks[s], tr[s], fn, N, N // 2, out=out, workspace=ws)
                q.metropolis_accept(R, S, ks[s], tr[s], out, u[s], fn, N, N // 2, acc=acc)
            accs[s].copy_(acc)

    def buffers():
        return (R0.clone(), torch.zeros((W, 5, Np), dtype=torch.float32, device="cuda"),
                torch.empty((W, 2, 5), dtype=torch.float64, device="cuda"),
                torch.empty((W, 2, 2), dtype=torch.float64, device="cuda"),
                torch.empty(W, dtype=torch.int32, device="cuda"),
                torch.empty((N, W), dtype=torch.int32, device="cuda"))

    e = buffers()
    run(*e)
    g_bufs = buffers()
    warm = buffers()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        run(*warm)
    torch.cuda.current_stream().wait_stream(cs)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        run(*g_bufs)
    g_bufs[0].copy_(R0)
    g_bufs[1].zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(e[0], g_bufs[0]) and torch.equal(e[1], g_bufs[1]) and torch.equal(e[5], g_bufs[5])
    a = e[5].cpu().numpy()
    assert 0 < a.sum() < a.size


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_fused_metropolis_accept_equals_separate_calls(q, dtype):
    """qj2_metropolis_accept (decision inside the accept kernel) == qj2_eval's
    ratio -> qj2_metropolis -> qj2_accept, bitwise (same fp64 decision), over a
    few sweep moves; and the fused decisions equal the oracle's where clear."""
    N, W = 3000, 96
    L = qmcgen.cell_length(N)
    Np = qmcgen.padded_size(N, 4 if dtype == np.float32 else 2)
    fn = q.Functor.of(qmcgen.make_functor(5, L))
    ks, tr, u = qmcgen.make_sweep(5, W, N, L, dtype, 4)
    R = qmcgen.positions(5, np.arange(W), N, Np, L, dtype)
    Ra, Rb = dev(R), dev(R)
    Sa = torch.zeros((W, 5, Np), dtype=Ra.dtype, device="cuda")
    Sb = torch.zeros_like(Sa)
    for s in range(4):
        kd, td, ud = dev(ks[s]), dev(tr[s]), dev(u[s])
        out_a, rat = q.eval(Ra, kd, td, fn, N, N // 2, ratio=True)
        acc_a = q.metropolis(rat, ud, trial=1)
        q.accept(Ra, Sa, kd, td, acc_a, out_a, fn, N, N // 2, trial=1)
        out_b = q.eval(Rb, kd, td, fn, N, N // 2)
        acc_b = q.metropolis_accept(Rb, Sb, kd, td, out_b, ud, fn, N, N // 2)
        assert torch.equal(acc_a, acc_b)
        o = out_b.cpu().numpy()
        rho2 = np.exp(o[:, 1, 0] - o[:, 0, 0]) ** 2
        clear = np.abs(u[s] - rho2) > 1e-9 * rho2
        assert np.array_equal(acc_b.cpu().numpy()[clear], (u[s] < rho2)[clear].astype(np.int32))
    assert torch.equal(Ra, Rb) and torch.equal(Sa, Sb)


def test_fused_metropolis_accept_sharded_slices(q):
    """qj2_metropolis_accept on source-axis slices (each rank's call with
    i_offset; r_k = trial 0 replicated) equals the unsharded call."""
    N, W = 20000, 24
    L = qmcgen.cell_length(N)
    fn = q.Functor.of(qmcgen.make_functor(19, L))
    ks, tr, u = qmcgen.make_sweep(19, W, N, L, np.float32, 1)
    R = qmcgen.positions(19, np.arange(W), N, qmcgen.padded_size(N, 4), L, np.float32)
    Rd = dev(R)
    S0 = torch.zeros((W, 5, R.shape[2]), dtype=torch.float32, device="cuda")
    out = q.eval(Rd, dev(ks[0]), dev(tr[0]), fn, N, N // 2)
    Ru, Su = Rd.clone(), S0.clone()
    acc_u = q.metropolis_accept(Ru, Su, dev(ks[0]), dev(tr[0]), out, dev(u[0]), fn, N, N // 2)
    bounds = [0, 7001, 13333, N]
    Rs, Ss = [], []
    for a, b in zip(bounds[:-1], bounds[1:]):
        Np = qmcgen.padded_size(b - a, 4)
        Rl = torch.zeros((W, 3, Np), dtype=torch.float32, device="cuda")
        Rl[:, :, :b - a] = Rd[:, :, a:b]
        Sl = torch.zeros((W, 5, Np), dtype=torch.float32, device="cuda")
        acc = q.metropolis_accept(Rl, Sl, dev(ks[0]), dev(tr[0]), out, dev(u[0]), fn, N, N // 2, i_offset=a,
                                  n_local=b - a)
        assert torch.equal(acc, acc_u)
        Rs.append(Rl[:, :, :b - a]); Ss.append(Sl[:, :, :b - a])
    assert torch.equal(torch.cat(Rs, 2), Ru[:, :, :N]) and torch.equal(torch.cat(Ss, 2), Su[:, :, :N])
