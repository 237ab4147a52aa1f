"""Development probe: XS vs XS2 (and repeat runs) on a 20,000-trial slice of config X: max relative
difference and determinism.  Not part of the product."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1412_4556_b200 import ara, synth  # noqa: E402

cfg = synth.Config.load("X")
elts = synth.make_elts(cfg)
N, K = 20_000, cfg.kmin
ids = torch.empty(N * K, dtype=torch.int32, device="cuda")
synth.yet_ids_device(ids.data_ptr(), cfg.seed, cfg.catalog_size, 0, N * K, torch.cuda.current_stream().cuda_stream)
ctx = ara.context_for_config(cfg, elts)
out = {}
for name, v in (("XS", 5), ("XS_again", 5), ("XS2", 6), ("XS2_again", 6), ("XS32", 7), ("lane", 1)):
    ctx.ara_set_option(ara.ARA_OPT_STREAM, v)
    y = torch.zeros((1, N), dtype=torch.float64, device="cuda")
    ctx.ara_run(ids, y, events_per_trial=K, num_trials=N)
    ctx.ara_check()
    out[name] = y.cpu().numpy()[0]
    print(name, ctx.ara_kernel_name(), flush=True)
b = out["XS"]
for k, v in out.items():
    d = np.abs(v - b)
    rel = d / np.maximum(np.abs(b), 1e-300)
    print(k, "differ:", int((v != b).sum()), "max abs", float(d.max()), "max rel", float(rel[b != 0].max() if (b != 0).any() else 0))
