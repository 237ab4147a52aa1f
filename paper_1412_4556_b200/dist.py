"""Trial sharding across GPUs: one process per GPU, contiguous trial blocks, NCCL YLT all-gather.

Trials are independent ("embarrassingly parallel"; one trial per thread, PAPER.md:199;
the paper decomposes the workload across GPU instances).  Rank g of G owns trials
[floor(g N / G), floor((g+1) N / G)) and a full replica of the (small) ELT tables.  The only exchange
is the YLT all-gather needed for the GLOBAL PML/TVaR quantiles: every rank's
[layers][shard] block is padded to shard_cap, gathered with one all_gather_into_tensor, and the
padding is removed by ara_unshard (device memcpy2D) -- no torch compute on the data path.

The shard arithmetic here is pure index bookkeeping and is tested with gloo on CPU
(tests/test_dist.py); the device steps are libara calls.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def shard_starts(num_trials: int, world: int) -> List[int]:
    """starts[g] = floor(g * N / G), g = 0..G (contiguous, sizes differ by at most one)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    return [(g * num_trials) // world for g in range(world + 1)]


def shard_range(num_trials: int, world: int, rank: int) -> Tuple[int, int]:
    s = shard_starts(num_trials, world)
    return s[rank], s[rank + 1]


def shard_cap(num_trials: int, world: int) -> int:
    s = shard_starts(num_trials, world)
    return max(s[g + 1] - s[g] for g in range(world))


def unshard_plan(starts: Sequence[int], cap: int, num_layers: int):
    """The copies ara_unshard performs, as (src_offset, dst_offset, length) in elements, for a
    gathered buffer [G][num_layers][cap] -> [num_layers][N].  Used by the CPU tests to check the
    bookkeeping the device function implements."""
    G = len(starts) - 1
    N = starts[-1]
    plan = []
    for g in range(G):
        cnt = starts[g + 1] - starts[g]
        for l in range(num_layers):
            plan.append(((g * num_layers + l) * cap, l * N + starts[g], cnt))
    return plan


def gather_ylt(local_ylt, num_trials: int, group=None):
    """All-gather per-rank YLT shards ([layers][shard] CUDA float64) into the full [layers][N] YLT on
    every rank.  One NCCL all_gather_into_tensor plus ara_unshard."""
    import torch
    import torch.distributed as dist

    from . import ara

    world = dist.get_world_size(group)
    L = local_ylt.shape[0]
    starts = shard_starts(num_trials, world)
    cap = shard_cap(num_trials, world)
    if local_ylt.shape[1] == cap and local_ylt.is_contiguous():
        send = local_ylt
    else:
        send = torch.empty((L, cap), dtype=local_ylt.dtype, device=local_ylt.device)
        send[:, :local_ylt.shape[1]].copy_(local_ylt)  # plumbing: pad the send buffer (D2D copy)
    recv = torch.empty((world, L, cap), dtype=local_ylt.dtype, device=local_ylt.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(recv.view(-1), send.reshape(-1), group=group)
    else:  # gloo (testing several ranks on one GPU): the same gather through host memory
        host = torch.empty(world * L * cap, dtype=local_ylt.dtype)
        dist.all_gather_into_tensor(host, send.reshape(-1).cpu(), group=group)
        recv.view(-1).copy_(host)
    full = torch.empty((L, num_trials), dtype=local_ylt.dtype, device=local_ylt.device)
    ara.ara_unshard(recv, world, cap, L, starts, full)
    return full
