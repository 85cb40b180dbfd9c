"""A/B of warp-per-walker kernel variants (QJ2_WARP) on one C4 wave shape:
256 instances x 1024 walkers of N = 6144 (fp32); CUDA events, best of 5."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_02645_b200 as q  # noqa: E402
import qmcgen  # noqa: E402
cfg = qmcgen.CONFIGS["C4"]
n_inst = 256
R = torch.empty((n_inst * cfg.W, 3, cfg.Np), dtype=torch.float32, device="cuda")
for j in range(n_inst):
    q.gen_positions(cfg.seed + j, cfg.W, cfg.N, cfg.Np, cfg.L, torch.float32, out=R[j * cfg.W:(j + 1) * cfg.W])
k = np.concatenate([qmcgen.make_k(cfg.seed + j, cfg.W, cfg.N) for j in range(n_inst)])
rt = np.concatenate([qmcgen.make_trials(cfg.seed + j, np.arange(cfg.W), qmcgen.make_k(cfg.seed + j, cfg.W, cfg.N),
                                        cfg.N, cfg.L, np.float32) for j in range(n_inst)])
kd, td = torch.from_numpy(k).cuda(), torch.from_numpy(rt).cuda()
fn = q.Functor.of(qmcgen.make_functor(cfg.seed, cfg.L, cfg.m))
out = torch.empty((n_inst * cfg.W, 1, 5), dtype=torch.float64, device="cuda")
ws = q.Workspace(0)
gb = n_inst * cfg.W * (cfg.N - 1) * 12 / 1e9
for v in (sys.argv[1:] or ["default", "p2m3"]):
    os.environ.pop("QJ2_WARP", None)
    if v != "default":
        os.environ["QJ2_WARP"] = v
    for _ in range(2):
        q.eval(R, kd, td, fn, cfg.N, cfg.n_up, out=out, workspace=ws)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); q.eval(R, kd, td, fn, cfg.N, cfg.n_up, out=out, workspace=ws); b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"{v}: {best:.3f} ms {gb / best * 1e3:.0f} GB/s", flush=True)
