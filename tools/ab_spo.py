"""A/B timing of the NEXT-4 SPO kernel variants on the S1 workload (80^3 x 384
orbitals, 65,536 walkers, vgh + ratio): QJ2_SPO=ldg (LDG kernel) and
QJ2_SPO_SMEM_KB (ring budget per CTA of the TMA kernel).  CUDA events, best
of 10.  Usage: python tools/ab_spo.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_02645_b200 as q  # noqa: E402
import qmcgen  # noqa: E402

cfg = qmcgen.SPO_CONFIGS["S1"]
coef = q.gen_spo_table(cfg.seed, cfg.nx, cfg.ny, cfg.nz, cfg.n_orb, cfg.ld)
tab = q.SpoTable(coef, cfg.n_orb, cfg.L)
pos = torch.from_numpy(qmcgen.spo_positions(cfg.seed, cfg.W, cfg.L)).cuda()
A = torch.from_numpy(qmcgen.make_ainv_rows(cfg.seed, cfg.W, cfg.n_orb)).cuda()
out = torch.empty((cfg.W, 5), dtype=torch.float64, device="cuda")
res = {}
VARIANTS = [("tma220", {"QJ2_SPO_SMEM_KB": "220"}), ("tma110", {"QJ2_SPO_SMEM_KB": "110"}),
            ("tma100", {"QJ2_SPO_SMEM_KB": "100"}), ("tma75", {"QJ2_SPO_SMEM_KB": "75"}),
            ("tma55", {"QJ2_SPO_SMEM_KB": "55"}), ("ldg", {"QJ2_SPO": "ldg"})]
for name, env in VARIANTS:
    for k in ("QJ2_SPO", "QJ2_SPO_SMEM_KB"):
        os.environ.pop(k, None)
    os.environ.update(env)
    for vgh in (True, False):
        for _ in range(3):
            q.spo_eval(tab, pos, vgh=vgh, Ainv=A, out=out)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            q.spo_eval(tab, pos, vgh=vgh, Ainv=A, out=out)
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        gb = cfg.W * (64 * cfg.n_orb * 4 + cfg.n_orb * 4 + 52) / 1e9
        res[f"{name}/{'vgh' if vgh else 'v'}"] = {"ms": best, "alg_GB_s": gb / best * 1e3}
        print(f"{name} {'vgh' if vgh else 'v'}: {best:.3f} ms {gb / best * 1e3:.0f} GB/s", file=sys.stderr, flush=True)
print(json.dumps(res))
