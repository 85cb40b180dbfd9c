"""Multi-GPU partitioning of the hot path.

One process per GPU (torchrun), NCCL via torch.distributed.  Two ways the path
shards, both from the paper's parallel structure:

* by instance / walker set (C4): walkers are independent (PAPER:1096-1108
  OpenMP over walkers, PAPER:1414-1416 MPI ranks hold disjoint walker sets);
  rank g takes instances [g*I/G, (g+1)*I/G); no collective on the data path.
* by source axis (C5): one walker set whose 1-by-N rows are split over ranks
  (the paper's proposed parallelism over electrons within a walker,
  PAPER:1665-1667).  Rank g evaluates its slice [g*N/G, (g+1)*N/G) with
  qj2_eval(i_offset=...) and the W*P*5 fp64 partial sums are combined with one
  all_reduce(SUM) -- the analog of the paper's per-generation MPI allreduce
  (PAPER:1423-1425).  Spin channel and self-exclusion use global indices, so
  the partials add up to the unsplit result.

The compute calls are injectable (eval_fn / ratio_fn) so the host-side
partition and combine logic is testable on CPU with a gloo process group; the
product default is the CUDA library (no CPU path).
"""
from __future__ import annotations

from typing import Callable, Iterable

import torch
import torch.distributed as dist


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block partition of range(n): rank gets [n*rank//world, n*(rank+1)//world)."""
    if world < 1 or not (0 <= rank < world) or n < 0:
        raise ValueError(f"bad partition n={n} rank={rank} world={world}")
    return n * rank // world, n * (rank + 1) // world


def instance_range(n_instances: int, rank: int, world: int) -> tuple[int, int]:
    """Instances owned by `rank` (C4)."""
    return shard_bounds(n_instances, rank, world)


def waves(first: int, count: int, max_resident: int) -> list[tuple[int, int]]:
    """Split [first, first+count) into consecutive waves of <= max_resident."""
    if max_resident < 1:
        raise ValueError("max_resident must be >= 1")
    out = []
    s = first
    while s < first + count:
        n = min(max_resident, first + count - s)
        out.append((s, n))
        s += n
    return out


def _default_eval():
    from . import eval as q_eval
    return q_eval


def _default_ratio():
    from . import ratio as q_ratio
    return q_ratio


def eval_sharded(R_local, k, r_trial, fn, n_total: int, n_up: int, i_offset: int, n_local: int, *,
                 group=None, V_cur=None, ratio: bool = False, out=None, ratio_out=None, workspace=None,
                 eval_fn: Callable | None = None, ratio_fn: Callable | None = None):
    """Source-axis split: partial (V, G, L) over this rank's slice, one
    all_reduce(SUM) over `group` (skipped when torch.distributed is not
    initialised or the group has one rank), then e^{dJ2} from the reduced sums.

    Returns out [W][P][5] (and ratio [W][P][2] if ratio=True)."""
    eval_fn = eval_fn or _default_eval()
    out = eval_fn(R_local, k, r_trial, fn, n_total, n_up, i_offset=i_offset, n_local=n_local,
                  out=out, workspace=workspace)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    if ratio:
        ratio_fn = ratio_fn or _default_ratio()
        return out, ratio_fn(out, V_cur=V_cur, ratio_out=ratio_out)
    return out


def _default(name):
    """An entry point of the CUDA library package (no CPU path)."""
    import importlib
    return getattr(importlib.import_module(__package__), name)


def sweep_step_sharded(R_local, state_local, k, r_trial, u, fn, n_total: int, n_up: int, i_offset: int,
                       n_local: int, *, group=None, out=None, ratio_out=None, acc=None, workspace=None,
                       accept_workspace=None, eval_fn: Callable | None = None, ratio_fn: Callable | None = None,
                       metropolis_fn: Callable | None = None, accept_fn: Callable | None = None):
    """One particle-by-particle move of every walker on a source-axis split
    (NEXT-2 at C5 scale; Alg. 1 L5-L9 for the J2 factor):

    1. eval_sharded with the P = 2 drift trials (r_k, r'_k): this rank's partial
       (V, G, L), one all_reduce(SUM), e^{dJ2} of trial 1 against trial 0;
    2. Metropolis u < rho^2 -- identical on every rank (the reduced sums and u
       are replicated), so no exchange of decisions;
    3. accept on this rank's slice of R and of the 5N state, with r_old = trial 0
       (= r_k, replicated: no exchange of positions); only the rank whose slice
       holds k commits r'_k and state_k (= the reduced out of trial 1).

    Returns (out [W][2][5], ratio [W][2][2], acc [W])."""
    out, ratio = eval_sharded(R_local, k, r_trial, fn, n_total, n_up, i_offset, n_local, group=group, ratio=True,
                              out=out, ratio_out=ratio_out, workspace=workspace, eval_fn=eval_fn,
                              ratio_fn=ratio_fn)
    metropolis_fn = metropolis_fn or _default("metropolis")
    accept_fn = accept_fn or _default("accept")
    acc = metropolis_fn(ratio, u, acc, trial=1)
    r_old = r_trial[:, 0, :].contiguous()
    accept_fn(R_local, state_local, k, r_trial, acc, out, fn, n_total, n_up, trial=1, i_offset=i_offset,
              n_local=n_local, r_old=r_old, workspace=accept_workspace)
    return out, ratio, acc


def gather_instances(local: torch.Tensor, counts: Iterable[int], group=None) -> torch.Tensor:
    """Concatenate per-rank results of the by-instance split on every rank
    (outside the timed region; e.g. per-instance checksums)."""
    counts = list(counts)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return local
    mx = max(counts)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in counts]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)
