"""The multi-GPU data path through product code, checked against the oracle.

Several ranks share the one GPU of the test box (NCCL cannot place two ranks on one device, so the
process group is gloo): each rank generates its trial block of the YET on the device, runs ara_run on
it, then dist.gather_ylt (padded all-gather + ara_unshard, the same code NCCL runs through) assembles
the full YLT on every rank, and rank 0 reads PML/TVaR with ara_pml_tvar.  The assembled YLT and the
metrics are compared with the CPU oracle over the whole (unsharded) YET: bitwise in the integer
regime (T), and bitwise against the single-process GPU run plus within the north_star tolerance of the
oracle in the real regime (V, ragged trials; P slice, stream kernel)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
from ara_testutil import within_tol
from paper_1412_4556_b200 import synth

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, num_trials, q):
    import torch.distributed as tdist

    from paper_1412_4556_b200 import ara
    from paper_1412_4556_b200 import dist as adist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.Config.load(name)
        N = num_trials or cfg.num_trials
        elts = synth.make_elts(cfg)
        ctx = ara.context_for_config(cfg, elts, device=0)
        t0, t1 = adist.shard_range(N, world, rank)
        dev = torch.device("cuda:0")
        L = len(cfg.layers)
        local = torch.empty((L, t1 - t0), dtype=torch.float64, device=dev)
        if cfg.fixed_length:  # device-generated YET shard (the bench's path)
            K = cfg.kmin
            ids = torch.empty((t1 - t0) * K, dtype=torch.int32, device=dev)
            synth.yet_ids_device(ids.data_ptr(), cfg.seed, cfg.catalog_size, t0 * K, (t1 - t0) * K,
                                 torch.cuda.current_stream().cuda_stream)
            ctx.ara_run(ids, local, events_per_trial=K, num_trials=t1 - t0)
        else:
            y = synth.make_yet(cfg, t0, t1)
            ids = torch.from_numpy(y.event_ids.view(np.int32)).to(dev)
            off = torch.from_numpy(y.offsets.view(np.int64)).to(dev)
            ctx.ara_run(ids, local, offsets=off, num_trials=t1 - t0)
        ctx.ara_check()
        full = adist.gather_ylt(local, N)
        torch.cuda.synchronize()
        if rank == 0:
            rps = synth.return_periods(N)
            pml, tvar = ara.ara_pml_tvar(full[0], rps)
            q.put((full.cpu().numpy(), pml, tvar, ctx.ara_kernel_name()))
        ctx.close()
        tdist.barrier()
    finally:
        tdist.destroy_process_group()


def _run(world, name, num_trials=0):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, num_trials, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    return got


@pytest.mark.parametrize("world", [2, 3])
def test_gather_ylt_integer_regime_bitwise_vs_oracle(cuda_device, world):
    cfg = synth.Config.load("T")
    y, pml, tvar, kern = _run(world, "T")
    want = oracle.ylt_for(cfg, synth.make_elts(cfg), synth.make_yet(cfg))
    rps = synth.return_periods(cfg.num_trials)
    assert kern.startswith("ara_presence_kernel"), kern  # the default for the paper-shaped layers
    assert np.array_equal(y, want)
    assert np.array_equal(pml, oracle.pml(want[0], rps)) and np.array_equal(tvar, oracle.tvar(want[0], rps))


@pytest.mark.parametrize("world,name,n", [(3, "V", 0), (2, "P", 20_000)])
def test_gather_ylt_real_regime_vs_oracle(cuda_device, world, name, n):
    cfg = synth.Config.load(name)
    elts = synth.make_elts(cfg)
    y, pml, tvar, _ = _run(world, name, n)
    N = n or cfg.num_trials
    want = oracle.ylt_for(cfg, elts, synth.make_yet(cfg, 0, N))
    assert y.shape == want.shape
    assert np.all(within_tol(y, want))
    rps = synth.return_periods(N)
    assert np.all(within_tol(pml, oracle.pml(want[0], rps))) and np.all(within_tol(tvar, oracle.tvar(want[0], rps)))
    # the sharded run equals a single-process run bitwise (trial-local summation order)
    y1, pml1, tvar1, _ = _run(1, name, n)
    assert np.array_equal(y, y1) and np.array_equal(pml, pml1) and np.array_equal(tvar, tvar1)


def test_bench_multi_rank_flow_completes(cuda_device):
    """bench.py under torchrun with two ranks (gloo on the one GPU): the sharded step -- per-rank run,
    YLT all-gather, PML/TVaR replayed on rank 0 -- completes and rank 0 prints one JSON line.  (A rank-0-only
    replay of the whole step once ran the all-gather on one rank and hung the job.)"""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"), "--gpus", "2", "--config",
           "T", "--steps", "3", "--warmup", "3", "--dist-backend", "gloo", "--no-e2e", "--no-cpu-baseline", "--no-cold"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and "error" not in d
