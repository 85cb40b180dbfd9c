"""The multi-rank path with the real CUDA library (-m gpu; one B200).

Only one GPU is available, so the ranks share cuda:0 and the process group is
gloo (NCCL refuses two ranks on one device); every rank runs the product's own
per-rank code -- paper_1708_02645_b200.parallel with the CUDA library, no oracle
injected -- and the combine is a real torch.distributed all_reduce over CUDA
tensors.  The ranks' kernels never wait on one another (the exchange is the
host-side collective), so sharing the device changes timing, not results.
Checked against the unsplit oracle:
* eval_sharded: the source-axis split of one instance at world 2 and 3 (uneven
  slices, rank-local generation with i_offset), PAPER:1665-1667;
* sweep_step_sharded: one particle-by-particle move (eval P = 2 -> all_reduce ->
  Metropolis -> accept on each slice), PAPER:1414-1426;
* bench.py under torchrun with 2 ranks (C5 source split with the all-reduce,
  C4 by instance): dist_init, barriers, max-over-ranks timing, rank-local input
  generation, per-rank waves; the line is a functional check, not a number.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import qmcgen

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
THREADS = os.cpu_count() or 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _eval_worker(rank, world, port, case, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1708_02645_b200 as qj
        from paper_1708_02645_b200 import parallel
        N, W, seed = case
        L = qmcgen.cell_length(N)
        a, b = parallel.shard_bounds(N, rank, world)
        Np = qmcgen.padded_size(b - a, 32)
        R = qj.gen_positions(seed, W, b - a, Np, L, torch.float32, i_offset=a)    # rank-local generation
        k = qmcgen.make_k(seed, W, N)
        rt = qmcgen.make_trials(seed, np.arange(W), k, N, L, np.float32, P=2, mode="drift")
        fn = qmcgen.make_functor(seed, L)
        out, ratio = parallel.eval_sharded(R, torch.from_numpy(k).cuda(), torch.from_numpy(rt).cuda(), fn, N, N // 2,
                                           a, b - a, ratio=True)
        torch.cuda.synchronize()
        q.put((rank, out.cpu().numpy(), ratio.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def _spawn(target, world, args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_eval_sharded_with_the_cuda_library(world):
    N, W, seed = 100_003, 48, 31
    res = _spawn(_eval_worker, world, ((N, W, seed),))
    L = qmcgen.cell_length(N)
    R = qmcgen.positions(seed, np.arange(W), N, N, L, np.float32)
    k = qmcgen.make_k(seed, W, N)
    rt = qmcgen.make_trials(seed, np.arange(W), k, N, L, np.float32, P=2, mode="drift")
    fn = qmcgen.make_functor(seed, L)
    orc, absout, _ = oracle.eval_j2(R, k, rt, fn, N, N // 2, threads=THREADS)
    for rank, out, ratio in res:
        assert np.array_equal(out, res[0][1])        # every rank holds the same reduced sums
        assert oracle.normalized_error(out, orc, absout, fn).max() <= 1e-5, rank
        dj = orc[:, 1, 0] - orc[:, 0, 0]
        assert np.all(ratio[:, 0, 0] == 0.0)
        assert np.max(np.abs(ratio[:, 1, 0] - dj) / np.maximum(absout[:, :, 0].max(1), 1.0)) <= 2e-5


def _sweep_worker(rank, world, port, case, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1708_02645_b200 import parallel
        N, W, seed = case
        L = qmcgen.cell_length(N)
        a, b = parallel.shard_bounds(N, rank, world)
        R = qmcgen.positions(seed, np.arange(W), N, N, L, np.float32)
        Np = qmcgen.padded_size(b - a, 32)
        Rl = np.zeros((W, 3, Np), np.float32)
        Rl[:, :, :b - a] = R[:, :, a:b]
        S0 = np.random.default_rng(seed).normal(size=(W, 5, N)).astype(np.float32)   # the update is additive
        Sl = np.zeros((W, 5, Np), np.float32)
        Sl[:, :, :b - a] = S0[:, :, a:b]
        ks, tr, u = qmcgen.make_sweep(seed, W, N, L, np.float32, 1)
        Rd, Sd = torch.from_numpy(Rl).cuda(), torch.from_numpy(Sl).cuda()
        fn = qmcgen.make_functor(seed, L)
        out, ratio, acc = parallel.sweep_step_sharded(Rd, Sd, torch.from_numpy(ks[0]).cuda(),
                                                      torch.from_numpy(tr[0]).cuda(), torch.from_numpy(u[0]).cuda(),
                                                      fn, N, N // 2, a, b - a)
        torch.cuda.synchronize()
        q.put((rank, a, b, acc.cpu().numpy(), Rd.cpu().numpy()[:, :, :b - a], Sd.cpu().numpy()[:, :, :b - a]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sweep_step_sharded_with_the_cuda_library(world):
    N, W, seed = 20_001, 24, 37
    res = _spawn(_sweep_worker, world, ((N, W, seed),))
    L = qmcgen.cell_length(N)
    R = qmcgen.positions(seed, np.arange(W), N, N, L, np.float32)
    S0 = np.random.default_rng(seed).normal(size=(W, 5, N)).astype(np.float32)
    ks, tr, u = qmcgen.make_sweep(seed, W, N, L, np.float32, 1)
    fn = qmcgen.make_functor(seed, L)
    orc, _, _ = oracle.eval_j2(R, ks[0], tr[0], fn, N, N // 2, threads=THREADS)
    rho2 = np.exp(orc[:, 1, 0] - orc[:, 0, 0]) ** 2
    acc = res[0][3]
    for r in res:
        assert np.array_equal(r[3], acc)            # identical decisions on every rank (no exchange)
    clear = np.abs(u[0] - rho2) > 1e-6 * rho2
    assert np.array_equal(acc[clear], (u[0] < rho2)[clear].astype(np.int32))
    assert 0 < acc.sum() < W
    R2, S2, ab = oracle.accept(R, S0, ks[0], tr[0][:, 1], acc, fn, N, N // 2)
    for rank, a, b, _, Rl, Sl in res:
        assert np.array_equal(Rl.astype(np.float64), R2[:, :, a:b]), rank     # only the owner of k commits r'_k
        e = oracle.normalized_error_state(Sl, S2[:, :, a:b], np.nan_to_num(ab[:, :, a:b]), fn)
        assert e.max() <= 1e-5, (rank, e.max())


@pytest.mark.parametrize("config,extra", [("C5", []), ("C4", ["--c4-instances", "64"])])
def test_bench_under_torchrun_two_ranks(config, extra):
    """bench.py's N > 1 path with 2 ranks on this one GPU (gloo, --same-device):
    one JSON line from rank 0 with n_gpus = 2 and the configuration's scaling."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--config", config, "--dist-backend", "gloo", "--same-device", "--no-e2e", *extra]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 2
    assert d["scaling"] == "strong"             # a fixed total (one C5 instance, 4096 C4 instances) split by rank
    assert d["config"]["parallelism"].endswith("x2")
