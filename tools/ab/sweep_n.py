"""Time qj2_sweep across electron counts (one ordered sweep = N moves of W
walkers per launch) with the library QJ2_LIB points at (else the product
build): the A/B helper for the sweep kernel's thread/partner tiers.

    python tools/ab/sweep_n.py [--W 1024] [--N 256,512,768,1024] [--j1] [--reps 10]

Prints one JSON line per N: ms per sweep and ns per move-partner (N*W*N).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import qmcgen  # noqa: E402
import paper_1708_02645_b200 as q  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--W", type=int, default=1024)
    ap.add_argument("--N", default="256,384,512,640,768,1000,1024")
    ap.add_argument("--j1", action="store_true")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    q.device_check()
    for N in [int(x) for x in a.N.split(",")]:
        seed = 7 + N
        L = qmcgen.cell_length(N)
        Np = qmcgen.padded_size(N, 32)
        R = torch.from_numpy(qmcgen.positions(seed, np.arange(a.W), N, Np, L, np.float32)).cuda()
        fn = qmcgen.make_functor(seed, L, 8)
        n_up = N // 2
        S = torch.zeros((a.W, 5, Np), dtype=torch.float32, device="cuda")
        j1 = None
        if a.j1:
            ions, start = qmcgen.make_ions(seed, 64, 64, L, np.float32, n_species=2)
            fn1 = qmcgen.make_j1_functor(seed, L, n_species=2)
            j1 = (torch.from_numpy(ions).cuda(), start, fn1,
                  torch.zeros((a.W, 5, Np), dtype=torch.float32, device="cuda"))
        q.state_init(R, S, fn, N, n_up, j1=j1)
        ks, delta, u = qmcgen.make_sweep_moves(seed, a.W, N, N)
        ks, delta, u = (torch.from_numpy(x).cuda() for x in (ks, delta, u))
        acc = torch.zeros(ks.shape, dtype=torch.int32, device="cuda")
        for _ in range(2):
            q.sweep(R, S, ks, delta, u, fn, N, n_up, acc=acc, j1=j1)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(a.reps):
            q.sweep(R, S, ks, delta, u, fn, N, n_up, acc=acc, j1=j1)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / a.reps
        print(json.dumps({"lib": os.environ.get("QJ2_LIB", "product"), "N": N, "W": a.W, "j1": a.j1,
                          "ms_per_sweep": ms, "ns_per_move_partner": ms * 1e6 / (N * a.W * N),
                          "accept_rate": float((acc == 1).float().mean())}), flush=True)


if __name__ == "__main__":
    main()
