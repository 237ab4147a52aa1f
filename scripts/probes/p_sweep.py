"""Same-box comparison of every kernel family and launch shape on config P (bench.py's inputs): the
default presence kernel, its other warp counts, the warp-ring, per-lane-queue and candidate-mask kernels.
Kernel time per 1M-trial launch, two alternating passes.  Development/evidence script."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1412_4556_b200 import ara, synth  # noqa: E402

cfg = synth.Config.load(sys.argv[1] if len(sys.argv) > 1 else "P")
elts = synth.make_elts(cfg)
stream = torch.cuda.current_stream()
ctx = ara.context_for_config(cfg, elts, device=0, stream=stream)
N, K = cfg.num_trials, cfg.kmin
ids = torch.empty(N * K, dtype=torch.int32, device="cuda")
synth.yet_ids_device(ids.data_ptr(), cfg.seed, cfg.catalog_size, 0, N * K, stream.cuda_stream)
ylt = torch.empty((len(cfg.layers), N), dtype=torch.float64, device="cuda")
nv = ctx.ara_layer_info(0)["num_variants"]


def t(stream_v=0, variant=0):
    ctx.ara_set_option(ara.ARA_OPT_KERNEL, ara.KERNEL_PRESENCE)
    ctx.ara_set_option(ara.ARA_OPT_STREAM, stream_v)
    ctx.ara_set_option(ara.ARA_OPT_VARIANT, variant)
    for _ in range(2):
        ctx.ara_run(ids, ylt, events_per_trial=K, num_trials=N, stream=stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(10):
        ctx.ara_run(ids, ylt, events_per_trial=K, num_trials=N, stream=stream)
    b.record(stream)
    torch.cuda.synchronize()
    ctx.ara_check()
    return ctx.ara_kernel_name(), a.elapsed_time(b) / 10


res = {}
for rep in range(2):
    for sv, v in [(0, i) for i in range(nv)] + [(1, 0), (2, 0), (3, 0), (4, 0), (9, 0), (10, 0)]:
        name, ms = t(sv, v)
        res.setdefault(name, []).append(round(ms, 4))
for name, ms in res.items():
    print(json.dumps({"kernel": name, "launch_ms": ms}), flush=True)
