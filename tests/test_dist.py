"""Multi-process trial sharding on CPU (gloo, world size 2 and 3): the shard arithmetic and the
gather/unshard bookkeeping reproduce the single-process YLT bitwise.  Per-rank compute here is the
oracle (CPU test harness); on the GPU the same plan is executed by ara_run + NCCL + ara_unshard."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1412_4556_b200 import dist as adist
from paper_1412_4556_b200 import synth


def test_shard_starts_cover_exactly():
    for N in (1, 7, 1000, 1_000_000, 8_000_000):
        for G in (1, 2, 3, 4, 8):
            s = adist.shard_starts(N, G)
            assert s[0] == 0 and s[-1] == N and all(b >= a for a, b in zip(s, s[1:]))
            sizes = [b - a for a, b in zip(s, s[1:])]
            assert max(sizes) - min(sizes) <= 1 and adist.shard_cap(N, G) == max(sizes)


def test_unshard_plan_is_a_permutation():
    for N, G, L in ((10, 3, 2), (1000, 8, 1), (7, 4, 3)):
        s, cap = adist.shard_starts(N, G), adist.shard_cap(N, G)
        seen = np.zeros(L * N, int)
        for src, dst, n in adist.unshard_plan(s, cap, L):
            assert src + n <= G * L * cap
            seen[dst:dst + n] += 1
        assert np.all(seen == 1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.Config.load(name)
    elts = synth.make_elts(cfg)
    t0, t1 = adist.shard_range(cfg.num_trials, world, rank)
    yet = synth.make_yet(cfg, t0, t1)           # each rank generates only its own shard
    local = oracle.ylt_for(cfg, elts, yet, threads=2)
    cap = adist.shard_cap(cfg.num_trials, world)
    L = len(cfg.layers)
    send = torch.full((L, cap), -1.0, dtype=torch.float64)
    send[:, :t1 - t0] = torch.from_numpy(local)
    recv = torch.empty((world * L * cap,), dtype=torch.float64)
    dist.all_gather_into_tensor(recv, send.reshape(-1))
    full = np.empty(L * cfg.num_trials)
    r = recv.numpy()
    for src, dst, n in adist.unshard_plan(adist.shard_starts(cfg.num_trials, world), cap, L):
        full[dst:dst + n] = r[src:src + n]
    if rank == 0:
        q.put(full.reshape(L, cfg.num_trials))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,name", [(2, "T"), (3, "V")])
def test_gloo_sharded_ylt_equals_single_process(world, name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = synth.Config.load(name)
    want = oracle.ylt_for(cfg, synth.make_elts(cfg), synth.make_yet(cfg))
    assert np.array_equal(got, want)
