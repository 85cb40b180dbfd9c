"""Shared comparison of qj2_sweep against the sweep oracle (test helper, not a
test module).

The GPU sweep runs on device copies; the oracle (oracle.sweep, pinned in
tests/test_oracle_sweep.py) replays the same moves from the same fp32 initial
state, forced onto the GPU's decisions so that both follow one trajectory, and
reports its own decisions and dJ.  Compared:
* decisions, where clear: |u - rho^2| > BAND * rho^2 with rho^2 = exp(2 dJ) of
  the oracle -- the GPU's dJ carries the fp32 state's rounding (U^2_k(R) is the
  stored fp32 entry, ~1e-6 relative), so decisions within that band of the
  threshold may legitimately differ;
* dJ: |dJ_gpu - dJ_orc| / max(A, 1) <= 1e-5 with A the from-scratch absolute
  sum of electron k's V terms (the scale of U^2_k);
* positions: bitwise (the proposal is fp32 on both sides);
* state: every entry within 1e-5 of the oracle's, normalized by the from-scratch
  absolute sums of the final configuration and the functor scale
  (oracle.normalized_error_state), and within 1e-5 of the final configuration's
  from-scratch state (the accumulated drift of the fp32 updates);
* J1 rows of moved electrons: normalized J1 error <= 1e-5.
"""
import os

import numpy as np
import torch

import oracle

BAND = 1e-3
THREADS = os.cpu_count() or 1


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check_sweep(q, R, state0, ks, delta, u, fn, N, n_up, *, j1=None, state_j1=None, walkers_state=None):
    """R [W][3][Np] fp32, state0 [W][5][Np] fp32 (consistent with R), ks [S][W],
    delta [S][W][3], u [S][W]; j1 = (ions fp32 [3][Np_ion], start, fn1) with
    state_j1 [W][5][Np] fp32 its initial rows.  walkers_state: walkers whose
    final state is checked against the O(N^2) from-scratch oracle (default all).
    Returns (acc, dj) of the GPU."""
    W = R.shape[0]
    Rd, Sd = dev(R), dev(state0)
    j1d = j1o = None
    if j1 is not None:
        ions, start, fn1 = j1
        S1d = dev(state_j1)
        j1d = (dev(ions), start, fn1, S1d)
        j1o = (ions.astype(np.float64), start, fn1, state_j1)
    acc, dj = q.sweep(Rd, Sd, dev(ks), dev(delta), dev(u), fn, N, n_up, j1=j1d)
    acc, dj = acc.cpu().numpy(), dj.cpu().numpy()
    R2, S2, own, dj_o, S1o = oracle.sweep(R, state0, ks, delta, u, fn, N, n_up, forced=acc, j1=j1o,
                                          threads=THREADS)
    valid = acc >= 0
    assert np.array_equal(own < 0, ~valid)
    rho2 = np.exp(2.0 * dj_o)
    clear = valid & (np.abs(u - rho2) > BAND * rho2)
    bad = np.argwhere(clear & (own != acc))
    assert bad.size == 0, f"decisions differ at (s, w) = {bad[:5].tolist()}"
    Rg = Rd.cpu().numpy()
    assert np.array_equal(Rg, R2), "positions differ"
    Sg = Sd.cpu().numpy()
    ws = range(W) if walkers_state is None else walkers_state
    dscale = np.ones(W)
    for w in ws:
        fresh, ab = oracle.j2_state(Rg[w].astype(np.float64), N, n_up, fn)
        dscale[w] = max(1.0, ab[0, :N].max())
        err = oracle.normalized_error_state(Sg[w][:, :N], S2[w][:, :N], ab[:, :N], fn).max()
        assert err <= 1e-5, (w, err)
        drift = oracle.normalized_error_state(Sg[w][:, :N], fresh[:, :N], ab[:, :N], fn).max()
        assert drift <= 1e-5, (w, drift)
    if walkers_state is None:
        assert np.max(np.abs(dj - dj_o)[valid] / np.broadcast_to(dscale, dj.shape)[valid]) <= 1e-5
    else:
        scale = np.maximum(np.abs(S2[:, 0, :N]).max(1), 1.0)
        assert np.max(np.abs(dj - dj_o)[valid] / np.broadcast_to(scale, dj.shape)[valid]) <= 1e-5
    if j1 is not None:
        S1g = j1d[3].cpu().numpy()
        moved = np.zeros((W, R.shape[2]), bool)
        for s in range(ks.shape[0]):
            a = acc[s] == 1
            moved[np.arange(W)[a], ks[s][a]] = True
        ions, start, fn1 = j1
        for w in range(W):
            e = np.nonzero(moved[w])[0]
            if e.size == 0:
                continue
            o1, a1 = oracle.eval_j1(ions.astype(np.float64), start, Rg[w][:, e].T.reshape(-1, 1, 3).astype(np.float64),
                                    fn1)
            err = oracle.normalized_error_j1(S1g[w][:, e].T.reshape(-1, 1, 5), S1o[w][:, e].T.reshape(-1, 1, 5),
                                             a1, fn1).max()
            assert err <= 1e-5, (w, err)
    return acc, dj
