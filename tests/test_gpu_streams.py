"""Calls on side streams (-m gpu): every entry point takes the caller's stream;
results on two concurrent side streams equal the default-stream results bitwise,
and the temporaries a call allocates for itself (workspaces, outputs) survive the
current stream reusing freed memory while the side-stream kernels still run."""
import numpy as np
import pytest
import torch

import qmcgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import paper_1708_02645_b200 as q
    q.device_check()
    return q


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _eval_inputs(seed, N, W, P=1):
    L = qmcgen.cell_length(N)
    Np = qmcgen.padded_size(N, 4)
    R = qmcgen.positions(seed, np.arange(W), N, Np, L, np.float32)
    k = qmcgen.make_k(seed, W, N)
    rt = qmcgen.make_trials(seed, np.arange(W), k, N, L, np.float32, P=P)
    return dev(R), dev(k), dev(rt), qmcgen.make_functor(seed, L)


def _churn():
    """Allocate and overwrite on the current stream (reuses freed blocks at once)."""
    for _ in range(4):
        torch.full((1 << 24,), 3.0e38, dtype=torch.float32, device="cuda")


def test_eval_on_two_side_streams(q):
    # 3 CTA tiles per walker: the call allocates a workspace (partials + counters)
    cases = [_eval_inputs(90 + i, 500000, 8, P=2) for i in range(2)]
    ref = [q.eval(R, k, rt, fn, 500000, 250000, ratio=True) for R, k, rt, fn in cases]
    torch.cuda.synchronize()
    ref = [(o.cpu(), r.cpu()) for o, r in ref]
    s = [torch.cuda.Stream(), torch.cuda.Stream()]
    got = []
    for rep in range(3):
        got = [q.eval(R, k, rt, fn, 500000, 250000, ratio=True, stream=s[i])
               for i, (R, k, rt, fn) in enumerate(cases)]
        _churn()
    torch.cuda.synchronize()
    for (o, r), (go, gr) in zip(ref, got):
        assert torch.equal(o, go.cpu()) and torch.equal(r, gr.cpu())


def test_sweep_on_two_side_streams(q):
    N, W = 768, 64
    L = qmcgen.cell_length(N)
    Np = qmcgen.padded_size(N, 32)
    fn = qmcgen.make_functor(95, L)
    runs = []
    for i in range(2):
        R = dev(qmcgen.positions(96 + i, np.arange(W), N, Np, L, np.float32))
        S = torch.zeros((W, 5, Np), dtype=torch.float32, device="cuda")
        q.state_init(R, S, fn, N, N // 2)
        ks, delta, u = (dev(a) for a in qmcgen.make_sweep_moves(97 + i, W, N, N))
        runs.append((R, S, ks, delta, u))
    torch.cuda.synchronize()
    ref = []
    for R, S, ks, delta, u in runs:
        R2, S2 = R.clone(), S.clone()
        acc, dj = q.sweep(R2, S2, ks, delta, u, fn, N, N // 2)
        ref.append((R2, S2, acc, dj))
    torch.cuda.synchronize()
    s = [torch.cuda.Stream(), torch.cuda.Stream()]
    got = []
    for i, (R, S, ks, delta, u) in enumerate(runs):
        R2, S2 = R.clone(), S.clone()
        torch.cuda.synchronize()
        acc, dj = q.sweep(R2, S2, ks, delta, u, fn, N, N // 2, stream=s[i])
        got.append((R2, S2, acc, dj))
    _churn()
    torch.cuda.synchronize()
    for a, b in zip(ref, got):
        for x, y in zip(a, b):
            assert torch.equal(x, y)


def test_spo_on_a_side_stream(q):
    tab = q.SpoTable(q.gen_spo_table(3, 24, 24, 24, 64, 64), 64, 9.0)
    W = 4096
    pos = dev(np.random.default_rng(5).uniform(0, 9.0, size=(W, 3)).astype(np.float32))
    A = dev(np.random.default_rng(6).normal(size=(W, 64)).astype(np.float32))
    ref = q.spo_eval(tab, pos, Ainv=A)
    torch.cuda.synchronize()
    ref = ref.cpu()
    s = torch.cuda.Stream()
    got = q.spo_eval(tab, pos, Ainv=A, stream=s)
    _churn()
    torch.cuda.synchronize()
    assert torch.equal(ref, got.cpu())
