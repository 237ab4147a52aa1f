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


class YltGather:
    """All-gather of per-rank YLT shards into the full [layers][N] YLT, with every buffer allocated once
    (the step itself allocates nothing): ara_run writes straight into the padded send buffer when the
    shard fills it, one NCCL all_gather_into_tensor, then ara_unshard (device memcpy2D) drops the
    padding.  `local` is the [layers][shard] view a rank's ara_run should write into."""

    def __init__(self, num_layers: int, num_trials: int, device, group=None):
        import torch
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.N = num_trials
        self.L = num_layers
        self.starts = shard_starts(num_trials, self.world)
        self.cap = shard_cap(num_trials, self.world)
        self.n_local = self.starts[self.rank + 1] - self.starts[self.rank]
        self.nccl = dist.get_backend(group) == "nccl"
        self.send = torch.zeros((num_layers, self.cap), dtype=torch.float64, device=device)
        self.recv = torch.empty((self.world, num_layers, self.cap), dtype=torch.float64, device=device)
        self.full = torch.empty((num_layers, num_trials), dtype=torch.float64, device=device)
        # ara_run's output: the send buffer itself when one layer fills it exactly, else a separate tensor
        direct = num_layers == 1 or self.n_local == self.cap
        self.local = self.send[:, :self.n_local] if (direct and num_layers == 1) else (
            self.send if direct else torch.empty((num_layers, self.n_local), dtype=torch.float64, device=device))
        self._host = None if self.nccl else torch.empty(self.world * num_layers * self.cap, dtype=torch.float64)

    def gather(self, stream=None):
        """Assemble self.full from every rank's self.local (stream-ordered; no allocation)."""
        import torch.distributed as dist

        from . import ara
        if self.local.data_ptr() != self.send.data_ptr():
            self.send[:, :self.n_local].copy_(self.local)  # pad the send rows (multi-layer, ragged shards)
        if self.nccl:
            dist.all_gather_into_tensor(self.recv.view(-1), self.send.view(-1), group=self.group)
        else:  # gloo (several ranks sharing one GPU in tests): the same gather through host memory
            dist.all_gather_into_tensor(self._host, self.send.view(-1).cpu(), group=self.group)
            self.recv.view(-1).copy_(self._host)
        ara.ara_unshard(self.recv, self.world, self.cap, self.L, self.starts, self.full, stream=stream)
        return self.full


_GATHERERS = {}


def gather_ylt(local_ylt, num_trials: int, group=None):
    """All-gather per-rank YLT shards ([layers][shard] CUDA float64) into the full [layers][N] YLT on
    every rank: one NCCL all_gather_into_tensor plus ara_unshard, through a cached YltGather (buffers
    allocated on the first call for a given shape)."""
    key = (local_ylt.shape[0], num_trials, local_ylt.device, id(group))
    g = _GATHERERS.get(key)
    if g is None:
        g = _GATHERERS[key] = YltGather(local_ylt.shape[0], num_trials, local_ylt.device, group)
    if local_ylt.data_ptr() != g.local.data_ptr():
        g.local.copy_(local_ylt) if g.local.shape == local_ylt.shape else g.send[:, :local_ylt.shape[1]].copy_(local_ylt)
    return g.gather()
