"""Benchmark of the ARA hot path (BASELINE.json metric: "ms per 1M-trial ARA run; ELT lookups/s and %
HBM roofline at 1/2/4/8 B200").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config P] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (one process per GPU, NCCL)

A step = one whole ARA run over the config's YET (BASELINE.json configs[1] "paper-shaped" by default:
1M trials x 1000 events x 16 ELTs): ara_run over every layer (YET stream -> row gathers -> FT1/FT2 ->
cumulative sum -> FT3 -> YLT), the NCCL YLT all-gather when N > 1, and PML/TVaR at the return periods
for every layer.  Trials are split in contiguous blocks over the ranks (strong scaling of the fixed
1M-trial run).  Inputs are device resident (the YET is generated in HBM by the seeded generator)
when the timed region starts; the ELT tables are built before it (ara_create, timed separately).
The YET (4 GB) is larger than L2, so no L2 flush is needed between steps; the 128 MB table is meant
to stay L2-resident (that is the design) -- a cold-L2 figure is reported beside it.

Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle (the reference arm for this
tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "ms per 1M-trial ARA run; ELT lookups/s and % HBM roofline at 1/2/4/8 B200"
UNIT = "ms/1M-trial run"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="P")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", type=int, default=None)
    ap.add_argument("--kernel", default=None, choices=["presence", "dense"], help="force the ARA kernel kind")
    ap.add_argument("--block", type=int, default=None)
    ap.add_argument("--bps", type=int, default=None)
    ap.add_argument("--l2-policy", type=int, default=None)
    ap.add_argument("--filter", type=int, default=None, choices=[-1, 0, 1],
                    help="ARA_OPT_FILTER: exact filter stage of the record presence kernel (-1 auto)")
    ap.add_argument("--stream", type=int, default=None,
                    help="ARA_OPT_STREAM: 0 = presence kernel for fixed-length trials, 1..3 = stream kernel variant")
    ap.add_argument("--prefetch", type=int, default=None, choices=[-1, 0, 1], help="ARA_OPT_PREFETCH")
    ap.add_argument("--round-min", type=int, default=None, help="ARA_OPT_ROUND_MIN (lane kernel round trigger)")
    ap.add_argument("--trial-order", type=int, default=None, choices=[0, 1], help="ARA_OPT_TRIAL_ORDER")
    ap.add_argument("--fused", type=int, default=None, choices=[0, 1], help="ARA_OPT_FUSED (multi-layer single pass)")
    ap.add_argument("--eager", action="store_true", help="issue the step's calls one by one (no captured plan)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cold", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="launch-shape sweep (E8); extra JSON lines to stderr")
    ap.add_argument("--cpu-sample", type=int, default=65536, help="trials in the cpu_baseline sample")
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no e2e/cold/cpu legs")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: exercise the multi-rank flow with several ranks sharing one GPU (testing only)")
    ap.add_argument("--study", action="store_true",
                    help="Section IV.B data-structure study (interleaved / independent / sorted ELTs); JSON lines to stderr")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region (B200_PROFILING.md clocks line).

    NVML is polled in-process every 5 ms from a thread started before the warm-up (so no tool start-up
    lands inside the timed region); only samples between mark_start() and mark_end() are reported.
    Falls back to `nvidia-smi -lms 10` when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.rows = []  # (time, sm_mhz, max_mhz, reasons bitmask or names)
        self.t0 = self.t1 = None
        self.stop = threading.Event()
        self.proc = None
        self.nvml = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.nvml = pynvml

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((time.perf_counter(), float(sm), float(mx), int(rs)))
                    except Exception:  # noqa: BLE001
                        pass
                    self.stop.wait(0.005)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.nvml = None
            try:
                q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                     "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
                self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                              "-lms", "10", "-i", str(self.index)], stdout=subprocess.PIPE,
                                             stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=self._read, daemon=True)
                self.t.start()
            except Exception:  # noqa: BLE001
                self.proc = None
        return self

    def _read(self):
        names = list(self.REASONS)
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6 and parts[0].replace(".", "").isdigit():
                bits = sum(self.REASONS[n] for n, v in zip(names, parts[2:]) if v.lower() == "active")
                self.rows.append((time.perf_counter(), float(parts[0]), float(parts[1]), bits))

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_end(self):
        self.t1 = time.perf_counter()

    def close(self):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        inside = [r for r in self.rows if self.t0 is not None and self.t1 is not None and self.t0 <= r[0] <= self.t1]
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        bits = 0
        for r in inside:
            bits |= r[3]
        return {"sm_mhz": float(np.median([r[1] for r in inside])), "sm_max_mhz": max(r[2] for r in inside),
                "reasons": sorted(n for n, b in self.REASONS.items() if bits & b), "samples": len(inside),
                "source": "nvml" if self.nvml else "nvidia-smi"}


def host_cpu():
    """lscpu model and topology of the host running the oracle."""
    info = {}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            info[k.strip()] = v.strip()
    except Exception:  # noqa: BLE001
        pass
    return {"model": info.get("Model name"), "sockets": info.get("Socket(s)"),
            "cores_per_socket": info.get("Core(s) per socket"), "threads_per_core": info.get("Thread(s) per core"),
            "online_cpus": info.get("On-line CPU(s) list"), "affinity_cpus": len(os.sched_getaffinity(0))}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ============================================================================ reference arm (CPU oracle)
def run_reference(args):
    import oracle
    from paper_1412_4556_b200 import synth
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = synth.Config.load(args.config)
    elts = synth.make_elts(cfg)
    cores = oracle.default_threads()
    sample = max(1, min(cfg.num_trials, 2048 if cfg.catalog_size <= 2_000_000 else 256))
    rps = synth.return_periods(sample)
    times = []
    for i in range(args.warmup + args.steps):
        stride = cfg.num_trials // sample
        trials = (np.arange(sample) * stride + (i % max(1, stride))) % cfg.num_trials
        yet = synth.make_yet_trials(cfg, trials)
        t0 = time.perf_counter()
        y = oracle.ylt_for(cfg, elts, yet, threads=cores)
        for l in range(len(cfg.layers)):
            if rps:
                oracle.pml(y[l], rps)
                oracle.tvar(y[l], rps)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    per_step = float(np.mean(times))
    value = per_step * 1e3 * 1e6 / sample
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.description}", "num_trials": cfg.num_trials,
                   "events_per_trial": [cfg.kmin, cfg.kmax], "layers": len(cfg.layers),
                   "elts_per_layer": len(cfg.layers[0].elts), "catalog": cfg.catalog_size,
                   "parallelism": f"oracle threads={cores}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "host": host_cpu(),
                         "extrapolation": cfg.num_trials / sample,
                         "sample": f"{sample} evenly spaced trials per step of {cfg.num_trials}; value extrapolated "
                                   f"x{cfg.num_trials / sample:g} to the full run"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ============================================================================ our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_1412_4556_b200 import ara, synth
    from paper_1412_4556_b200 import dist as adist

    world, rank, local = dist_env()
    if world > 1:
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    cfg = synth.Config.load(args.config)
    L = len(cfg.layers)
    N = cfg.num_trials
    t0, t1 = adist.shard_range(N, world, rank)
    n_local = t1 - t0
    elts = synth.make_elts(cfg)

    # ---- preprocessing stage: tables (timed separately)
    torch.cuda.synchronize()
    c0 = time.perf_counter()
    ctx = ara.context_for_config(cfg, elts, device=dev.index, stream=stream)
    create_ms = (time.perf_counter() - c0) * 1e3
    if args.kernel is not None:
        ctx.ara_set_option(ara.ARA_OPT_KERNEL, ara.KERNEL_DENSE if args.kernel == "dense" else ara.KERNEL_PRESENCE)
    if args.variant is not None:
        ctx.ara_set_option(ara.ARA_OPT_VARIANT, args.variant)
    if args.block is not None:
        ctx.ara_set_option(ara.ARA_OPT_BLOCK_THREADS, args.block)
    if args.bps is not None:
        ctx.ara_set_option(ara.ARA_OPT_BLOCKS_PER_SM, args.bps)
    if args.l2_policy is not None:
        ctx.ara_set_option(ara.ARA_OPT_L2_POLICY, args.l2_policy)
    if args.filter is not None:
        ctx.ara_set_option(ara.ARA_OPT_FILTER, args.filter)
    if args.stream is not None:
        ctx.ara_set_option(ara.ARA_OPT_STREAM, args.stream)
    if args.prefetch is not None:
        ctx.ara_set_option(ara.ARA_OPT_PREFETCH, args.prefetch)
    if args.round_min is not None:
        ctx.ara_set_option(ara.ARA_OPT_ROUND_MIN, args.round_min)
    if args.trial_order is not None:
        ctx.ara_set_option(ara.ARA_OPT_TRIAL_ORDER, args.trial_order)
    if args.fused is not None:
        ctx.ara_set_option(ara.ARA_OPT_FUSED, args.fused)
    info = [ctx.ara_layer_info(l) for l in range(L)]

    # ---- this rank's YET shard, generated in HBM
    if cfg.fixed_length:
        K = cfg.kmin
        q0, q1 = t0 * K, t1 * K
        offsets_d = None
        offsets_h = None
    else:
        K = 0
        off = synth.trial_offsets(cfg.seed, N, cfg.kmin, cfg.kmax)
        q0, q1 = int(off[t0]), int(off[t1])
        offsets_h = (off[t0:t1 + 1] - np.uint64(q0)).astype(np.uint64)
        offsets_d = torch.from_numpy(offsets_h.view(np.int64)).to(dev)
    n_ids = q1 - q0
    ids = torch.empty(n_ids, dtype=torch.int32, device=dev)
    synth.yet_ids_device(ids.data_ptr(), cfg.seed, cfg.catalog_size, q0, n_ids, sp)
    rps = synth.return_periods(N)
    m = len(rps)
    met = torch.zeros((L, 2, max(m, 1)), dtype=torch.float64, device=dev)  # per layer: PML row, TVaR row
    met_h = torch.empty((L, 2, max(m, 1)), dtype=torch.float64, pin_memory=True)
    gat = adist.YltGather(L, N, dev) if world > 1 else None
    ylt_local = gat.local if gat is not None else torch.empty((L, n_local), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()

    # ara_run over every layer is captured once (ara_plan_create: one CUDA graph, launch attributes and
    # folds set up beforehand), so the timed loop issues one graph launch per step for it; the CUDA events
    # around that launch time the ARA kernels alone.  --eager issues ara_run directly.
    plan = None
    mplan = [None]  # captured PML/TVaR (ara_metrics_plan_create), set up after the correctness gate
    if not args.eager:
        plan = ctx.ara_plan_create(ids, ylt_local, [], None, None, offsets=offsets_d, events_per_trial=K,
                                   num_trials=n_local, stream=stream)

    def step(evs=None):
        """One pass of the hot path: ara_run (all layers) -> [all-gather] -> PML/TVaR per layer (on rank 0
        when sharded), results copied to pinned host memory on the same stream (no host round trip)."""
        nvtx = torch.cuda.nvtx  # host-side ranges (an nsys/ncu timeline shows the step's phases)
        if evs is not None:
            evs[0].record(stream)
        nvtx.range_push("ara_run")
        if plan is not None:
            plan.launch(stream=stream)
        else:
            ctx.ara_run(ids, ylt_local, offsets=offsets_d, events_per_trial=K, num_trials=n_local, stream=stream)
        nvtx.range_pop()
        if evs is not None:
            evs[1].record(stream)
        nvtx.range_push("gather+pml_tvar")
        full = gat.gather(stream=stream) if world > 1 else ylt_local
        if m and (world == 1 or rank == 0):
            if mplan[0] is not None:  # one graph launch: every layer's PML/TVaR into the host-copied rows
                mplan[0].launch(stream=stream)
            else:
                for l in range(L):  # results straight into the rows copied to the host (no device-side copies)
                    ara.ara_pml_tvar_device(full[l], rps, met[l, 0], met[l, 1], stream=stream)
        nvtx.range_pop()
        if evs is not None:
            evs[2].record(stream)
        if m and (world == 1 or rank == 0):
            met_h.copy_(met, non_blocking=True)
        return full

    # ---- correctness gate + cpu baseline (oracle on a bounded sample of this rank's trials)
    full = step()
    ctx.ara_check(stream)
    torch.cuda.synchronize()
    for l in range(L if m and (world == 1 or rank == 0) else 0):  # the captured/async metrics equal the sync API's
        p_sync, t_sync = ara.ara_pml_tvar(full[l], rps, stream=stream)
        if not (np.array_equal(p_sync, met_h[l, 0].numpy()) and np.array_equal(t_sync, met_h[l, 1].numpy())):
            print(json.dumps({"error": f"layer {l}: ara_pml_tvar_device != ara_pml_tvar"}), flush=True)
            sys.exit(3)
    if m and (world == 1 or rank == 0) and not args.eager:  # the captured metric step, checked bit for bit
        mplan[0] = ara.ara_metrics_plan_create(full, rps, met[:, 0], met[:, 1], out_stride=2 * met.shape[2],
                                               stream=stream)
        ref_h = met_h.clone()
        met.zero_()
        mplan[0].launch(stream=stream)  # (not step(): a sharded step's gather is a collective of all ranks)
        met_h.copy_(met, non_blocking=True)
        torch.cuda.synchronize()
        if not torch.equal(met_h, ref_h):
            print(json.dumps({"error": "captured metric step != ara_pml_tvar_device"}), flush=True)
            sys.exit(3)
    cpu = None
    if not args.profile and not args.no_cpu_baseline:
        import oracle
        cores = oracle.default_threads()
        sample = min(n_local, args.cpu_sample)
        trials = t0 + (np.arange(sample, dtype=np.int64) * n_local) // sample
        yet_s = synth.make_yet_trials(cfg, trials)
        c0 = time.perf_counter()
        y_or = oracle.ylt_for(cfg, elts, yet_s, threads=cores)
        for l in range(L):
            if len(synth.return_periods(sample)):
                oracle.pml(y_or[l], synth.return_periods(sample))
                oracle.tvar(y_or[l], synth.return_periods(sample))
        cpu_s = time.perf_counter() - c0
        got = ylt_local[:, torch.from_numpy(trials - t0).to(dev)].cpu().numpy()
        tol = np.maximum(1e-6 * np.abs(y_or), 1e-3)
        err = np.abs(got - y_or)
        bad = int(np.sum(err > tol))
        nz = np.abs(y_or) > 0
        parity = {"sampled_trials": int(sample), "max_abs_err": float(err.max()) if err.size else 0.0,
                  "max_rel_err": float((err[nz] / np.abs(y_or[nz])).max()) if np.any(nz) else 0.0,
                  "bitwise_equal": int(np.sum(got == y_or)), "tolerance": "|gpu - oracle| <= max(1e-6 |oracle|, 1e-3)"}
        if bad:
            print(json.dumps({"error": f"parity gate failed: {bad} of {got.size} sampled YLT values outside "
                                       f"1e-6 rel / 1e-3 abs of the oracle"}), flush=True)
            sys.exit(3)
        cpu = {"value": cpu_s * 1e3 * 1e6 / sample, "unit": UNIT, "cores": cores, "kind": "oracle",
               "host": host_cpu(), "extrapolation": 1e6 / sample,
               "sample": f"{sample} evenly spaced trials of rank {rank}'s shard (YLT + PML/TVaR on the sample), "
                         f"{cpu_s:.2f} s wall; "
                         + ("the whole workload, no extrapolation" if sample >= n_local else
                            f"value extrapolated x{1e6 / sample:.3g} to 1M trials")
                         + "; the same sample gates GPU parity "
                         f"(0 of {got.size} outside tolerance)",
               "parity_checked": int(got.size), "parity": parity}

    clk = ClockSampler(dev.index).start()  # started before the warm-up: no tool start-up inside the timed region
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    # ---- timed region (warm: the table stays L2-resident; the 4 GB YET streams from HBM)
    kev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk.mark_start()
    start.record(stream)
    for i in range(args.steps):
        step(kev[i])
    end.record(stream)
    torch.cuda.synchronize()
    clk.mark_end()
    clk.close()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = start.elapsed_time(end)
    kern_ms = float(np.mean([a.elapsed_time(b) for a, b, _ in kev]))
    post_ms = float(np.mean([b.elapsed_time(c) for _, b, c in kev]))  # gather + PML/TVaR
    step_ms_list = [kev[i][0].elapsed_time(kev[i + 1][0]) for i in range(len(kev) - 1)]
    t = torch.tensor([total_ms, kern_ms, post_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, kern_ms, post_ms = float(t[0]), float(t[1]), float(t[2])
    ms_per_step = total_ms / args.steps
    ctx.ara_check(stream)

    # ---- cold-L2 variant: flush L2 (write 512 MB) before each step, untimed
    cold_ms = None
    if not args.profile and not args.no_cold:
        scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        cold = []
        for i in range(min(args.steps, 5)):
            scratch.fill_(i & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step()
            b.record(stream)
            torch.cuda.synchronize()
            cold.append(a.elapsed_time(b))
        del scratch
        ct = torch.tensor([float(np.mean(cold))], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ct, op=dist.ReduceOp.MAX)
        cold_ms = float(ct[0])

    # ---- end to end through the public API with HOST buffers (ara_run_host)
    e2e = None
    if not args.profile and not args.no_e2e:
        host_ids = torch.empty(n_ids, dtype=torch.int32, pin_memory=True)
        host_ids.copy_(ids)
        host_ylt = torch.empty((L, n_local), dtype=torch.float64, pin_memory=True)
        dev_ylt = torch.empty((L, n_local), dtype=torch.float64, device=dev)

        def e2e_step():
            ctx.ara_run_host(host_ids, host_ylt, offsets=offsets_h, events_per_trial=K, num_trials=n_local,
                             stream=stream)
            dev_ylt.copy_(host_ylt, non_blocking=True)  # the metrics read the YLT on the device
            full = adist.gather_ylt(dev_ylt, N) if world > 1 else dev_ylt
            return [ara.ara_pml_tvar(full[l], rps, stream=stream) for l in range(L)] if rps else []

        e2e_step()
        e2e_step()
        ne = min(args.steps, 7)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ne)]
        for a, b in evs:
            a.record(stream)
            e2e_step()
            b.record(stream)
        torch.cuda.synchronize()
        per = [a.elapsed_time(b) for a, b in evs]
        # median over the steps: one slow PCIe window (seen once on a freshly booted box) should not
        # stand for the path; every step's time is reported beside it
        et = torch.tensor([float(np.median(per))], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e_ms = float(et[0])
        h2d = n_ids * 4 + (offsets_h.nbytes if offsets_h is not None else 0) + L * n_local * 8
        d2h = L * n_local * 8 + L * len(rps) * 16
        e2e = {"value": e2e_ms * 1e6 / N, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e2e_ms, "step_ms": [round(x, 3) for x in per], "stat": "median of %d steps" % ne,
               "path": "ara_run_host (pinned host YET streamed in 256 MB batches, copy/compute "
                                              "overlapped) + ara_pml_tvar (result to host)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (one launch per layer)
    occ = n_ids  # occurrences on this rank per layer pass
    row_bytes = [max(32, i["row_stride"]) for i in info]  # sector-rounded row bytes
    launch_ms = kern_ms / L
    peak, peak_src = peaks()
    kernel_full = ctx.ara_kernel_name()  # the kernel the timed runs launched
    kernel_name = kernel_full.split("<")[0]
    sparse_path = kernel_name in ("ara_presence_kernel", "ara_stream_kernel", "ara_lane_kernel", "ara_mask_kernel")
    # compulsory HBM bytes of one presence-kernel launch: the YET ids (4 B per occurrence), the YLT
    # row (8 B per trial), and one read of every table row that holds a loss plus the bitmap
    present_rows = [ctx.ara_layer_stats(l)["present_rows"] for l in range(L)]
    comp_bytes = float(np.mean([4.0 * occ + 8.0 * n_local + pr * rb + (cfg.catalog_size + 1) / 8.0
                                for pr, rb in zip(present_rows, row_bytes)]))
    dense_bytes = float(np.mean([occ * (4 + rb) for rb in row_bytes]))  # 4 B id + row sectors
    if kernel_name == "ara_fused_kernel":
        # one launch streams the YET once for every layer: YET ids + every layer's YLT row, present rows
        # and bitmap
        launch_ms = kern_ms
        alg_bytes_launch = 4.0 * occ + sum(8.0 * n_local + pr * rb + (cfg.catalog_size + 1) / 8.0
                                           for pr, rb in zip(present_rows, row_bytes))
        alg_note = ("fused multi-layer pass (one launch for %d layers): algorithmic bytes = compulsory HBM traffic: "
                    "4 B YET id per occurrence once + per layer 8 B YLT per trial, its rows holding a loss and its "
                    "presence bitmap (DESIGN.md 'Roofline')" % L)
    elif sparse_path:
        alg_bytes_launch = comp_bytes
        alg_note = ("algorithmic bytes = compulsory HBM traffic: 4 B YET id per occurrence + 8 B YLT per trial + "
                    "one read of each table row holding a loss (%d rows x %d B) + the presence bitmap; rows of "
                    "events absent from every ELT are all-zero and never fetched (DESIGN.md 'Roofline')"
                    % (present_rows[0], row_bytes[0]))
    else:
        alg_bytes_launch = dense_bytes
        alg_note = "algorithmic bytes = occurrences x (4 B id + %d B sector-rounded row), SURVEY.md 8(d)" % row_bytes[0]
    achieved = alg_bytes_launch / (launch_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"ncu_{cfg.name}.json")
    if os.path.exists(prof):
        with open(prof) as f:
            pj = json.load(f)
        if pj.get("variant") == kernel_full and world == 1:  # the capture is of the N = 1 launch
            traffic = pj.get("dram_bytes_per_launch")

    # ---- the dense direct-access kernel (every occurrence gathers its full row), timed beside
    dense = None
    presence_leg = None
    pres_ylt = None
    if not args.profile and args.variant is None and sparse_path:
        ctx.ara_set_option(ara.ARA_OPT_KERNEL, ara.KERNEL_DENSE)
        for _ in range(2):
            ctx.ara_run(ids, ylt_local, offsets=offsets_d, events_per_trial=K, num_trials=n_local, stream=stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        nd = 5
        for _ in range(nd):
            ctx.ara_run(ids, ylt_local, offsets=offsets_d, events_per_trial=K, num_trials=n_local, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        dms = a.elapsed_time(b) / nd / L
        dense = {"kernel": ctx.ara_layer_info(0)["variant"], "launch_ms": dms,
                 "achieved_GBps": dense_bytes / (dms * 1e-3) / 1e9, "frac": dense_bytes / (dms * 1e-3) / 1e9 / peak,
                 "alg_bytes_per_launch": dense_bytes,
                 "note": "SURVEY.md 8(d) definition: occurrences x (4 B id + sector-rounded row); table gathers are "
                         "served mostly from DRAM (ncu: L2 hit ~36%)"}
        ctx.ara_set_option(ara.ARA_OPT_KERNEL, ara.KERNEL_AUTO)
        ctx.ara_check(stream)
    # ---- the layer-outer passes (Algorithm 1's loop order), timed beside the fused pass
    outer_leg = None
    if not args.profile and L > 1 and kernel_name == "ara_fused_kernel":
        ref_ylt = ylt_local.clone()
        ctx.ara_set_option(ara.ARA_OPT_FUSED, 0)
        for _ in range(2):
            ctx.ara_run(ids, ylt_local, offsets=offsets_d, events_per_trial=K, num_trials=n_local, stream=stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(3):
            ctx.ara_run(ids, ylt_local, offsets=offsets_d, events_per_trial=K, num_trials=n_local, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        diff = (ylt_local - ref_ylt).abs()
        over = diff > torch.maximum(1e-12 * ref_ylt.abs(), torch.full_like(ref_ylt, 1e-6))
        rel = float((diff / ref_ylt.abs().clamp_min(1e-300))[ref_ylt.abs() > 1e-3].max()) if bool((ref_ylt.abs() > 1e-3).any()) else 0.0
        first_bad = torch.nonzero(over)[:3].tolist()
        outer_leg = {"kernel": ctx.ara_kernel_name(), "ms_all_layers": a.elapsed_time(b) / 3,
                     "fused_ms_all_layers": kern_ms, "max_rel_diff_vs_fused": rel,
                     "elements_beyond_1e-12": int(over.sum()), "first": first_bad,
                     "first_values": [[float(ref_ylt[i, j]), float(ylt_local[i, j])] for i, j in first_bad],
                     "note": "one pass per layer (PAPER.md:104-105) vs one fused pass over the YET (SURVEY.md N1)"}
        ctx.ara_set_option(ara.ARA_OPT_FUSED, 1)
        ctx.ara_check(stream)
    elif not args.profile and L > 1 and cfg.fixed_length:  # the product is layer-outer: time the fused pass
        ref_ylt = ylt_local.clone()
        ctx.ara_set_option(ara.ARA_OPT_FUSED, 1)
        for _ in range(2):
            ctx.ara_run(ids, ylt_local, offsets=offsets_d, events_per_trial=K, num_trials=n_local, stream=stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(3):
            ctx.ara_run(ids, ylt_local, offsets=offsets_d, events_per_trial=K, num_trials=n_local, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        diff = (ylt_local - ref_ylt).abs()
        over = diff > torch.maximum(1e-12 * ref_ylt.abs(), torch.full_like(ref_ylt, 1e-6))
        outer_leg = {"kernel": ctx.ara_kernel_name(), "fused_ms_all_layers": a.elapsed_time(b) / 3,
                     "layer_outer_ms_all_layers": kern_ms, "elements_beyond_1e-12_vs_layer_outer": int(over.sum()),
                     "note": "SURVEY.md N1: one fused pass over the YET for all layers (ARA_OPT_FUSED=1) vs the "
                             "layer-outer product path (PAPER.md:104-105); the fused pass is the slower one here"}
        ctx.ara_set_option(ara.ARA_OPT_FUSED, 0)
        ctx.ara_check(stream)
    # ---- SURVEY N3 ablation: the precombined occurrence-net table o[e] (no ELT lookups at run time),
    # timed beside; its YLT must equal the product path's bit for bit (checked here)
    pre = None
    if not args.profile and args.variant is None and sparse_path:
        ctx.ara_run(ids, ylt_local, offsets=offsets_d, events_per_trial=K, num_trials=n_local, stream=stream)
        ref_ylt = ylt_local.clone()  # the product path's YLT
        # the round-1 presence kernel (stream kernel off), timed beside: its YLT must equal bit for bit
        if kernel_name in ("ara_stream_kernel", "ara_lane_kernel", "ara_mask_kernel"):
            ctx.ara_set_option(ara.ARA_OPT_STREAM, 0)
            ctx.ara_set_option(ara.ARA_OPT_FILTER, 0)  # the presence kernel itself (no exact scan filter)
            for _ in range(2):
                ctx.ara_run(ids, ylt_local, offsets=offsets_d, events_per_trial=K, num_trials=n_local, stream=stream)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(5):
                ctx.ara_run(ids, ylt_local, offsets=offsets_d, events_per_trial=K, num_trials=n_local, stream=stream)
            b.record(stream)
            torch.cuda.synchronize()
            presence_leg = {"kernel": ctx.ara_kernel_name(), "launch_ms": a.elapsed_time(b) / 5 / L,
                            "ylt_bitwise_equal": bool(torch.equal(ylt_local, ref_ylt)),
                            "max_rel_diff": float(((ylt_local - ref_ylt).abs() / ref_ylt.abs().clamp_min(1e-3)).max())}
            pres_ylt = ylt_local.clone()
            ctx.ara_set_option(ara.ARA_OPT_STREAM, 0 if args.stream is None else args.stream)
            ctx.ara_set_option(ara.ARA_OPT_FILTER, -1 if args.filter is None else args.filter)
        ctx.ara_set_option(ara.ARA_OPT_PRECOMBINED, 1)
        for _ in range(2):
            ctx.ara_run(ids, ylt_local, offsets=offsets_d, events_per_trial=K, num_trials=n_local, stream=stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        npc = 5
        for _ in range(npc):
            ctx.ara_run(ids, ylt_local, offsets=offsets_d, events_per_trial=K, num_trials=n_local, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        pms = a.elapsed_time(b) / npc / L
        # N3 is an ablation of the presence kernel: compare with its YLT (bitwise, same summation order)
        base = pres_ylt if pres_ylt is not None else ref_ylt
        same = bool(torch.equal(ylt_local, base))
        ctx.ara_set_option(ara.ARA_OPT_PRECOMBINED, 0)
        ctx.ara_check(stream)
        pre = {"launch_ms": pms, "ylt_bitwise_equal": same,
               "note": "SURVEY.md 8(f) N3 ablation: per-layer table o[e] = FT2(sum_j FT1(l_ej)) built once; a hit "
                       "gathers one 8-B value and does no FT1/FT2 work.  Exact for deterministic losses only; "
                       "performs no ELT lookups at run time, so it is not the headline"}
    lookups_exact = float(sum(len(l.elts) for l in cfg.layers)) * (
        N * cfg.kmin if cfg.fixed_length else float(synth.trial_offsets(cfg.seed, N, cfg.kmin, cfg.kmax)[-1]))
    value = ms_per_step * 1e6 / N
    # one ara_layer/presence launch per layer, one fused (cooperative) metric launch per layer and batch
    # of <= 16 return periods; the NCCL all-gather (N > 1) and ara_unshard's memcpy2D are not our kernels
    n_metric_launches = L * ((len(rps) + 15) // 16) if rps else 0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.description}", "num_trials": N,
                   "events_per_trial": [cfg.kmin, cfg.kmax], "layers": L, "elts_per_layer": len(cfg.layers[0].elts),
                   "catalog": cfg.catalog_size, "entries_per_elt": cfg.entries_per_elt, "regime": cfg.regime,
                   "parallelism": f"trial-sharded x{world}" + (
                       (" + NCCL YLT all-gather" if args.dist_backend == "nccl" else " + gloo YLT all-gather (host)")
                       if world > 1 else ""),
                   "l2": "no flush: inputs (YET %.1f GB) exceed L2; table L2-resident by design (cold_l2_ms beside)"
                         % (n_ids * 4 / 1e9),
                   "kernel": kernel_full, "storage": "fp32 ELT losses, fp64 terms/sums/YLT"},
        "trials_per_s": N / (ms_per_step * 1e-3),
        "elt_lookups_per_s": lookups_exact / (ms_per_step * 1e-3),
        "kernel_ms_per_step": kern_ms, "gather_metrics_ms_per_step": post_ms,
        "step_ms_min_median_max": [round(float(np.min(step_ms_list)), 4), round(float(np.median(step_ms_list)), 4),
                                   round(float(np.max(step_ms_list)), 4)] if step_ms_list else None,
        "create_ms": create_ms, "cold_l2_ms_per_step": cold_ms,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": kernel_name,
                     "alg_bytes_per_launch": alg_bytes_launch, "launch_ms": launch_ms,
                     "effective_GBps_68B": dense_bytes / (launch_ms * 1e-3) / 1e9,
                     "note": alg_note + f"; peak {peak_src}"},
        "dense_kernel": dense,
        "presence_kernel": presence_leg,
        "layer_outer_N1": outer_leg,
        "precombined_N3": pre,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": args.steps * (L + n_metric_launches),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)

    if args.sweep:
        info[0]["product_kernel"] = kernel_full
        sweep(ctx, ids, offsets_d, K, n_local, L, ylt_local, stream, info, occ)
    if args.study:
        study(ctx, cfg, ids, offsets_d, offsets_h, K, n_local, L, ylt_local, stream, occ, kern_ms)
    if world > 1:
        dist.destroy_process_group()


def study(ctx, cfg, ids, offsets_d, offsets_h, K, n_local, L, ylt_local, stream, occ, kern_ms):
    """PAPER.md:209-213 (Section IV.B): the same Algorithm 1 over three ELT representations.  Each layout
    runs a plain one-lane-per-occurrence kernel; the product kernels are listed beside for reference.
    The sorted/binary-search layout runs on a 1/16 trial subset and is scaled."""
    import torch

    from paper_1412_4556_b200 import ara
    J = sum(len(l.elts) for l in cfg.layers) / L
    for layout, name in ((ara.STUDY_INTERLEAVED, "interleaved"), (ara.STUDY_INDEPENDENT, "independent"),
                         (ara.STUDY_SORTED, "sorted+binary-search"), (ara.STUDY_HASH, "hash"),
                         (ara.STUDY_INDEX, "event->compact-row index")):
        n = n_local if layout != ara.STUDY_SORTED else max(1, n_local // 16)
        if offsets_d is None:
            sub_ids, sub_off = ids[: n * K], None
        else:
            sub_ids, sub_off = ids, offsets_d[: n + 1]
        ctx.ara_run_study(layout, sub_ids, ylt_local, offsets=sub_off, events_per_trial=K, num_trials=n, stream=stream)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        a.record(stream)
        for _ in range(reps):
            ctx.ara_run_study(layout, sub_ids, ylt_local, offsets=sub_off, events_per_trial=K, num_trials=n, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps * (n_local / n)
        print(json.dumps({"study": name, "ms_per_1M_trial_run": ms * 1e6 / n_local / 1.0,
                          "launch_ms_all_layers": ms, "lookups_per_s": occ * J * L / (ms * 1e-3),
                          "subset_trials": n}), file=sys.stderr, flush=True)
    print(json.dumps({"study": "product (presence/dense, ara_run)", "launch_ms_all_layers": kern_ms,
                      "lookups_per_s": occ * J * L / (kern_ms * 1e-3)}), file=sys.stderr, flush=True)


def sweep(ctx, ids, offsets_d, K, n_local, L, ylt_local, stream, info, occ):
    """Launch-shape sweep (the paper's threads-per-block study, E8): kernel time per
    (variant, block threads, blocks per SM, L2 policy)."""
    import torch

    from paper_1412_4556_b200 import ara
    rb = max(32, info[0]["row_stride"])
    if info[0].get("product_kernel", "").startswith(("ara_stream", "ara_lane", "ara_mask")):  # fixed-length-trial kernels
        for sv in (1, 4):
            for pf in (0, 1):
                for pol in (0, 1):  # here: the trial order (0 blocks, 1 interleaved)
                    ctx.ara_set_option(ara.ARA_OPT_STREAM, sv)
                    ctx.ara_set_option(ara.ARA_OPT_PREFETCH, pf)
                    ctx.ara_set_option(ara.ARA_OPT_TRIAL_ORDER, pol)
                    for _ in range(2):
                        ctx.ara_run(ids, ylt_local, offsets=None, events_per_trial=K, num_trials=n_local, stream=stream)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    for _ in range(5):
                        ctx.ara_run(ids, ylt_local, offsets=None, events_per_trial=K, num_trials=n_local, stream=stream)
                    b.record(stream)
                    torch.cuda.synchronize()
                    print(json.dumps({"sweep": ctx.ara_kernel_name(), "prefetch": pf, "trial_order": pol,
                                      "launch_ms": a.elapsed_time(b) / 5 / L}), file=sys.stderr, flush=True)
        ctx.ara_set_option(ara.ARA_OPT_PREFETCH, -1)
        ctx.ara_set_option(ara.ARA_OPT_TRIAL_ORDER, 1)
        ctx.ara_set_option(ara.ARA_OPT_STREAM, 0)  # then the presence kernel's own sweep
    nv = info[0]["num_variants"]
    presence = info[0]["variant"].startswith("ara_presence")
    for v in range(nv):
        # presence kernels fix their block size: sweep the next-trial prefetch instead of block threads
        for bt in ((0, 1) if presence else (128, 256)):
            for bps in (0,) if presence else (0, 2, 3, 4, 6, 8):
                for pol in (0, 1, 2):
                    try:
                        ctx.ara_set_option(ara.ARA_OPT_VARIANT, v)
                        if presence:
                            ctx.ara_set_option(ara.ARA_OPT_PREFETCH, bt)
                        else:
                            ctx.ara_set_option(ara.ARA_OPT_BLOCK_THREADS, bt)
                        ctx.ara_set_option(ara.ARA_OPT_BLOCKS_PER_SM, bps)
                        ctx.ara_set_option(ara.ARA_OPT_L2_POLICY, pol)
                    except ara.AraError:
                        continue
                    for _ in range(2):
                        ctx.ara_run(ids, ylt_local, offsets=offsets_d, events_per_trial=K, num_trials=n_local, stream=stream)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    for _ in range(5):
                        ctx.ara_run(ids, ylt_local, offsets=offsets_d, events_per_trial=K, num_trials=n_local, stream=stream)
                    b.record(stream)
                    torch.cuda.synchronize()
                    ms = a.elapsed_time(b) / 5 / L
                    print(json.dumps({"sweep": ctx.ara_layer_info(0)["variant"], ("prefetch" if presence else "block"): bt,
                                      "bps": bps, "l2_policy": pol,
                                      "launch_ms": ms, "eff_GBps": occ * (4 + rb) / ms / 1e6}), file=sys.stderr, flush=True)
    ctx.ara_set_option(ara.ARA_OPT_VARIANT, 0)
    if presence:
        ctx.ara_set_option(ara.ARA_OPT_PREFETCH, 0)  # the library default
    ctx.ara_set_option(ara.ARA_OPT_BLOCK_THREADS, 0)
    ctx.ara_set_option(ara.ARA_OPT_BLOCKS_PER_SM, 0)
    ctx.ara_set_option(ara.ARA_OPT_L2_POLICY, 0)
    ctx.ara_set_option(ara.ARA_OPT_STREAM, 1)


if __name__ == "__main__":
    main()
