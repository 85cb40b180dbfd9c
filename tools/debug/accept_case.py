"""Debug one randomized accept case (tests/test_gpu_randomized.py::test_accept_random)
by shift and id: per-entry normalized errors with the pair geometry behind them."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
os.environ["QJ2_RANDOM_SHIFT"] = sys.argv[1]
import test_gpu_randomized as t  # noqa: E402
import oracle  # noqa: E402
import qmcgen  # noqa: E402
import paper_1708_02645_b200 as q  # noqa: E402

want = sys.argv[2]
for c in t._accept_cases():
    cid = f"N{c['N']}-W{c['W']}-m{c['m']}-{'f64' if c['f64'] else 'f32'}"
    if cid != want:
        continue
    print(c)
    N, W, m, f64, seed, up_frac, p_acc = c["N"], c["W"], c["m"], c["f64"], c["seed"], c["up_frac"], c["p_acc"]
    dtype = np.float64 if f64 else np.float32
    L = qmcgen.cell_length(N)
    Np = qmcgen.padded_size(N, 2 if f64 else 4)
    R = qmcgen.positions(seed, np.arange(W), N, Np, L, dtype)
    k = qmcgen.make_k(seed, W, N)
    rt = qmcgen.make_trials(seed, np.arange(W), k, N, L, dtype)
    fn = qmcgen.make_functor(seed, L, m)
    rng = np.random.default_rng(seed)
    state = rng.normal(size=(W, 5, Np)).astype(dtype)
    state[:, :, N:] = 7.0
    acc = (rng.random(W) < p_acc).astype(np.int32)
    n_up = int(round(up_frac * N))
    Rd, Sd = t.dev(R), t.dev(state)
    out = q.eval(Rd, t.dev(k), t.dev(rt), fn, N, n_up)
    q.accept(Rd, Sd, t.dev(k), t.dev(rt), t.dev(acc), out, fn, N, n_up)
    Sg = Sd.cpu().numpy()
    R2, S2, ab = oracle.accept(R, state, k, rt[:, 0], acc, fn, N, n_up)
    err = oracle.normalized_error_state(Sg[:, :, :N], S2[:, :, :N], ab[:, :N] if ab.ndim == 2 else ab[:, :, :N], fn)
    print("L", L, "r_cut", fn.r_cut, "delta", fn.r_cut / fn.m, "k", k, "acc", acc, "n_up", n_up)
    for w in range(W):
        print("walker", w, "k", k[w], "acc", acc[w], "r_k", R[w, :, k[w]], "r'", rt[w, 0])
        for i in range(N):
            d_old = R[w, :, i].astype(np.float64) - R[w, :, k[w]]
            d_new = R[w, :, i].astype(np.float64) - rt[w, 0].astype(np.float64)
            d_old -= L * np.round(d_old / L)
            d_new -= L * np.round(d_new / L)
            print(f"  i={i} |r-r_k|={np.linalg.norm(d_old):.6g} |r-r'|={np.linalg.norm(d_new):.6g} "
                  f"err={err[w, :, i]} gpu={Sg[w, :, i]} orc={S2[w, :, i]} abs={ab[w, :, i]}")
