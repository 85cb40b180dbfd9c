"""Host-side multi-rank logic of paper_1708_02645_b200.parallel on CPU:
partition properties, and world-size-2 gloo runs of the source-axis split
(eval_sharded: per-rank partial sums + all_reduce + ratio) and of the
instance gather, with the per-rank compute injected from the oracle (CPU).
The per-rank CUDA kernel path itself is covered by the fake-shard GPU tests."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import qmcgen

# parallel.py imports the package lazily only for its default compute; import
# the module file directly so these CPU tests never need the CUDA library.
import importlib.util

_spec = importlib.util.spec_from_file_location(
    "qj2_parallel", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                 "paper_1708_02645_b200", "parallel.py"))
parallel = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(parallel)


def test_shard_bounds_partition():
    for n in (0, 1, 7, 4096, 4915200):
        for world in (1, 2, 3, 4, 8):
            b = [parallel.shard_bounds(n, r, world) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        parallel.shard_bounds(10, 2, 2)


def test_waves():
    w = parallel.waves(1024, 2048, 1000)
    assert w == [(1024, 1000), (2024, 1000), (3024, 48)]
    assert parallel.waves(0, 0, 5) == []


def _oracle_eval(R, k, rt, fn, n_total, n_up, i_offset=0, n_local=None, out=None, workspace=None):
    o, _, _ = oracle.eval_j2(R.numpy(), k.numpy(), rt.numpy(), fn, n_total, n_up,
                             i_offset=i_offset, n_local=n_local)
    t = torch.from_numpy(o)
    if out is not None:
        out.copy_(t)
        return out
    return t


def _numpy_ratio(out, V_cur=None, ratio_out=None):
    o = out.numpy()
    ref = V_cur.numpy()[:, None] if V_cur is not None else o[:, :1, 0]
    dj = o[:, :, 0] - ref
    return torch.from_numpy(np.stack([dj, np.exp(dj)], axis=-1))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N, W = 203, 6
        L = qmcgen.cell_length(N)
        R = qmcgen.positions(5, np.arange(W), N, 208, L, np.float64)
        k = qmcgen.make_k(5, W, N)
        rt = qmcgen.make_trials(5, np.arange(W), k, N, L, np.float64, P=2, mode="drift")
        fn = qmcgen.make_functor(5, L)
        a, b = parallel.shard_bounds(N, rank, world)
        Rl = np.zeros((W, 3, 208))
        Rl[:, :, :b - a] = R[:, :, a:b]
        out, rat = parallel.eval_sharded(torch.from_numpy(Rl), torch.from_numpy(k), torch.from_numpy(rt), fn,
                                         N, N // 2, a, b - a, ratio=True,
                                         eval_fn=_oracle_eval, ratio_fn=_numpy_ratio)
        full, absout, _ = oracle.eval_j2(R, k, rt, fn, N, N // 2)
        err = float(oracle.normalized_error(out.numpy(), full, absout, fn).max())
        dj = full[:, 1, 0] - full[:, 0, 0]
        rerr = float(np.max(np.abs(rat.numpy()[:, 1, 0] - dj)))
        # instance gather with unequal counts
        counts = [3, 2][:world] if world == 2 else [3]
        local = torch.full((counts[rank], 5), float(rank))
        g = parallel.gather_instances(local, counts)
        q.put((rank, err, rerr, g.numpy().tolist()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_source_split_allreduce_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, rerr, g in res:
        assert err < 1e-13, (rank, err)          # reduced partials == unsplit oracle
        assert rerr < 1e-12, (rank, rerr)
        assert g == [[0.0] * 5] * 3 + [[1.0] * 5] * 2
