"""A/B timing of the multi-trial (P > 1) eval kernel variants on the C3
instance (N = 614,400, W = 1024, fp32): QJ2_KERNEL selects the CTA kernel
variant (launch.cuh: ldg1, p3m2, tma323).  CUDA events, best of reps.
Usage: python tools/ab_multitrial.py [P ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_02645_b200 as q  # noqa: E402
import qmcgen  # noqa: E402

cfg = qmcgen.CONFIGS["C3"]
Ps = [int(a) for a in sys.argv[1:]] or [2, 4, 12]
variants = os.environ.get("AB_VARIANTS", "default,p3m2,ldg1").split(",")
R = q.gen_positions(cfg.seed, cfg.W, cfg.N, cfg.Np, cfg.L, torch.float32)
k = qmcgen.make_k(cfg.seed, cfg.W, cfg.N)
fn = q.Functor.of(qmcgen.make_functor(cfg.seed, cfg.L, cfg.m))
kd = torch.from_numpy(k).cuda()
res = {}
for P in Ps:
    rt = torch.from_numpy(qmcgen.make_trials(cfg.seed, np.arange(cfg.W), k, cfg.N, cfg.L, np.float32, P=P,
                                             mode="drift")).cuda()
    ws = q.Workspace(q.workspace_size(cfg.W, P, cfg.N, torch.float32))
    out = torch.empty((cfg.W, P, 5), dtype=torch.float64, device="cuda")
    ref = None
    for v in variants:
        os.environ.pop("QJ2_KERNEL", None)
        if v != "default":
            os.environ["QJ2_KERNEL"] = v
        for _ in range(3):
            q.eval(R, kd, rt, fn, cfg.N, cfg.n_up, out=out, workspace=ws)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            q.eval(R, kd, rt, fn, cfg.N, cfg.n_up, out=out, workspace=ws)
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        o = out.cpu().numpy()
        same = True if ref is None else float(np.max(np.abs(o - ref) / np.maximum(np.abs(ref), 1.0)))
        ref = o if ref is None else ref
        res[f"P{P}/{v}"] = {"ms": best, "items_per_s": cfg.W * P * (cfg.N - 1) / best * 1e3, "same_as_default": same}
        print(f"P={P} {v}: {best:.3f} ms", file=sys.stderr, flush=True)
print(json.dumps(res))
