"""Diagnose the end-to-end host path: ara_run_host timing with torch-pinned vs pageable YET buffers."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ARA_DEBUG"] = "1"
import numpy as np, torch
from paper_1412_4556_b200 import ara, synth
cfg = synth.Config.load("P")
elts = synth.make_elts(cfg)
ctx = ara.context_for_config(cfg, elts)
K, N = cfg.kmin, 250_000
n = N * K
d = torch.empty(n, dtype=torch.int32, device="cuda")
synth.yet_ids_device(d.data_ptr(), cfg.seed, cfg.catalog_size, 0, n, torch.cuda.current_stream().cuda_stream)
hp = torch.empty(n, dtype=torch.int32, pin_memory=True); hp.copy_(d)
print("is_pinned", hp.is_pinned())
yp = torch.empty((1, N), dtype=torch.float64, pin_memory=True)
for name, h, y in [("pinned", hp, yp), ("pinned-ids/np-ylt", hp, np.zeros((1, N))), ("pageable", hp.numpy().copy(), np.zeros((1, N)))]:
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        ctx.ara_run_host(h, y, events_per_trial=K, num_trials=N)
        dt = time.perf_counter() - t
        print(f"{name} rep{rep}: {dt*1e3:.1f} ms  -> {n*4/dt/1e9:.1f} GB/s", flush=True)
