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
        counts = [3, 2, 4][:world]
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


@pytest.mark.parametrize("world", [2, 3])
def test_source_split_allreduce_gloo(world):
    """C5's source-axis split at world 2 and 3 (unequal shards of N = 203)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
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
        counts = [3, 2, 4][:world]
        assert g == sum(([[float(r)] * 5] * counts[r] for r in range(world)), [])


# ---------------------------------------------------------------------------
# NEXT-2 at C5 scale: one PbyP move on a source-axis split (sweep_step_sharded)
# ---------------------------------------------------------------------------
def _numpy_metropolis(ratio, u, acc=None, trial=0):
    rho = ratio.numpy()[:, trial, 1]
    return torch.from_numpy((u.numpy() < rho * rho).astype(np.int32))


def _oracle_accept_slice(R_local, S_local, k, r_trial, acc, out, fn, n_total, n_up, trial=0, i_offset=0,
                         n_local=None, r_old=None, workspace=None):
    """CPU stand-in for qj2_accept on a slice with the kernel's semantics: the
    oracle's partner update on the slice's electrons (r_k from the caller's
    r_old), state_k = the reduced eval output of the accepted trial, R[:, k]
    committed by the owner."""
    W, _, Np = R_local.shape
    Rl, Sl = R_local.numpy(), S_local.numpy()
    a, b = i_offset, i_offset + n_local
    ro, rn = r_old.numpy(), r_trial.numpy()[:, trial]
    for w in range(W):
        if not acc[w]:
            continue
        kw = int(k[w])
        # a full-length stand-in row: the slice's electrons in place, r_k at k
        Rf = np.zeros((1, 3, n_total))
        Rf[0, :, a:b] = Rl[w, :, :n_local]
        Rf[0, :, kw] = ro[w]
        Sf = np.zeros((1, 5, n_total))
        Sf[0, :, a:b] = Sl[w, :, :n_local]
        _, S2, _ = oracle.accept(Rf, Sf, np.array([kw], np.int32), rn[w:w + 1], np.ones(1, np.int32), fn,
                                 n_total, n_up)
        Sl[w, :, :n_local] = S2[0, :, a:b]
        if a <= kw < b:
            Sl[w, :, kw - a] = out.numpy()[w, trial]
            Rl[w, :, kw - a] = rn[w]
    return R_local, S_local


def _sweep_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N, W = 150, 8
        L = qmcgen.cell_length(N)
        R = qmcgen.positions(9, np.arange(W), N, N, L, np.float64)
        fn = qmcgen.make_functor(9, L)
        state = np.stack([oracle.j2_state(R[w], N, N // 2, fn)[0] for w in range(W)])
        ks, tr, u = qmcgen.make_sweep(9, W, N, L, np.float64, 1)
        k, rt, uu = ks[0], tr[0], u[0]
        a, b = parallel.shard_bounds(N, rank, world)
        Rl = torch.from_numpy(np.ascontiguousarray(R[:, :, a:b]))
        Sl = torch.from_numpy(np.ascontiguousarray(state[:, :, a:b]))
        out, rat, acc = parallel.sweep_step_sharded(
            Rl, Sl, torch.from_numpy(k), torch.from_numpy(rt), torch.from_numpy(uu), fn, N, N // 2, a, b - a,
            eval_fn=_oracle_eval, ratio_fn=_numpy_ratio, metropolis_fn=_numpy_metropolis,
            accept_fn=_oracle_accept_slice)
        # unsplit reference: oracle eval, the same decision, oracle accept
        full, _, _ = oracle.eval_j2(R, k, rt, fn, N, N // 2)
        acc_ref = (uu < np.exp(full[:, 1, 0] - full[:, 0, 0]) ** 2).astype(np.int32)
        R2, S2, ab = oracle.accept(R, state, k, rt[:, 1], acc_ref, fn, N, N // 2)
        serr = float(oracle.normalized_error_state(Sl.numpy(), S2[:, :, a:b], np.nan_to_num(ab[:, :, a:b]),
                                                   fn).max())
        q.put((rank, acc.numpy().tolist(), acc_ref.tolist(), bool(np.array_equal(Rl.numpy(), R2[:, :, a:b])),
               serr))
    finally:
        dist.destroy_process_group()


def test_sweep_step_source_split_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_sweep_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    accs = [r[1] for r in res]
    assert accs[0] == accs[1] == res[0][2]          # identical decisions on every rank, = the unsplit oracle
    assert 0 < sum(accs[0]) < len(accs[0])
    for rank, _, _, r_ok, serr in res:
        assert r_ok, rank                            # positions: only the owner of k commits r'_k
        assert serr < 1e-12, (rank, serr)
