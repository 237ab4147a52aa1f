"""Development probe: cost of PML/TVaR inside a captured plan (graph) vs the eager per-call path, on P."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1412_4556_b200 import ara, synth  # noqa: E402

cfg = synth.Config.load("P")
elts = synth.make_elts(cfg)
s = torch.cuda.current_stream()
ctx = ara.context_for_config(cfg, elts, device=0, stream=s)
N, K = cfg.num_trials, cfg.kmin
ids = torch.empty(N * K, dtype=torch.int32, device="cuda")
synth.yet_ids_device(ids.data_ptr(), cfg.seed, cfg.catalog_size, 0, N * K, s.cuda_stream)
ylt = torch.empty((1, N), dtype=torch.float64, device="cuda")
rps = synth.return_periods(N)
pm = torch.zeros((1, len(rps)), dtype=torch.float64, device="cuda")
tv = torch.zeros_like(pm)
plain = ctx.ara_plan_create(ids, ylt, [], None, None, events_per_trial=K, num_trials=N, stream=s)
withm = ctx.ara_plan_create(ids, ylt, rps, pm, tv, events_per_trial=K, num_trials=N, stream=s)


def t(fn, reps=30):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for rep in range(2):
    tp = t(lambda: plain.launch(stream=s))
    tw = t(lambda: withm.launch(stream=s))
    te = t(lambda: (plain.launch(stream=s), ara.ara_pml_tvar_device(ylt[0], rps, pm[0], tv[0], stream=s)))
    tm = t(lambda: ara.ara_pml_tvar_device(ylt[0], rps, pm[0], tv[0], stream=s), 200)
    print(f"plan {tp:.4f} ms; plan+metrics in graph {tw:.4f} (metrics {1e3 * (tw - tp):.1f} us); "
          f"plan + eager metrics {te:.4f} (metrics {1e3 * (te - tp):.1f} us); eager metrics alone {1e3 * tm:.1f} us",
          flush=True)

# two graphs back to back (ARA plan, then the captured metric step) with and without an event between them
mplan = ara.ara_metrics_plan_create(ylt, rps, pm[0], tv[0], stream=s)
ev = torch.cuda.Event()
for rep in range(2):
    tp = t(lambda: plain.launch(stream=s))
    t2 = t(lambda: (plain.launch(stream=s), mplan.launch(stream=s)))
    t3 = t(lambda: (plain.launch(stream=s), ev.record(s), mplan.launch(stream=s)))
    tw = t(lambda: withm.launch(stream=s))
    print(f"two graphs {1e3 * (t2 - tp):.1f} us of metrics; with an event between {1e3 * (t3 - tp):.1f} us; "
          f"one graph {1e3 * (tw - tp):.1f} us", flush=True)
