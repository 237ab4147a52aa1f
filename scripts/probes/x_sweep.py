"""Development probe: config X kernel time per fixed-length-trial XS variant / round trigger / prefetch /
trial order, all on one box with bench.py's inputs.  Not part of the product."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1412_4556_b200 import ara, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "X"
cfg = synth.Config.load(name)
elts = synth.make_elts(cfg)
stream = torch.cuda.current_stream()
ctx = ara.context_for_config(cfg, elts, device=0, stream=stream)
N, K = cfg.num_trials, cfg.kmin
ids = torch.empty(N * K, dtype=torch.int32, device="cuda")
synth.yet_ids_device(ids.data_ptr(), cfg.seed, cfg.catalog_size, 0, N * K, stream.cuda_stream)
ylt = torch.empty((len(cfg.layers), N), dtype=torch.float64, device="cuda")


def t(**opt):
    for k, v in opt.items():
        ctx.ara_set_option(getattr(ara, "ARA_OPT_" + k.upper()), v)
    for _ in range(2):
        ctx.ara_run(ids, ylt, events_per_trial=K, num_trials=N, stream=stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(4):
        ctx.ara_run(ids, ylt, events_per_trial=K, num_trials=N, stream=stream)
    b.record(stream)
    torch.cuda.synchronize()
    ctx.ara_check()
    ms = a.elapsed_time(b) / 4
    print(json.dumps({"kernel": ctx.ara_kernel_name(), **opt, "launch_ms": round(ms, 3),
                      "ms_per_1M": round(ms * 1e6 / N, 3)}), flush=True)
    return ylt.clone()


base = t(stream=0, prefetch=-1, trial_order=1, round_min=24)
if os.environ.get("X_SWEEP_BASE_ONLY"):
    sys.exit(0)
for extra in [dict(stream=5), dict(stream=6), dict(stream=7), dict(stream=8),
              dict(stream=5, round_min=16), dict(stream=5, round_min=20), dict(stream=5, round_min=28),
              dict(stream=5, round_min=24, prefetch=0), dict(stream=5, prefetch=1, trial_order=0)]:
    y = t(**{**dict(stream=0, prefetch=-1, trial_order=1, round_min=24), **extra})
    if not torch.equal(y, base):
        print(json.dumps({"note": "YLT differs from the default run", **extra}), flush=True)
