"""Development probe: phase times of metrics_select (ARA_METRICS_TRACE) and per-call device time on 1M
values shaped like a YLT (zero years, capped years, a continuous body), and on uniform reals."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1412_4556_b200 import ara, synth  # noqa: E402

os.environ["ARA_METRICS_TRACE"] = "1"
rng = np.random.default_rng(5)
n = 1_000_000
rps = synth.return_periods(n)
cases = {
    "ylt_like": np.where(rng.random(n) < 0.25, 0.0, np.minimum(rng.lognormal(15, 1.0, n), 9e6)),
    "uniform": rng.random(n) * 1e9,
    "ties": np.floor(rng.exponential(1e6, n)) * (rng.random(n) > 0.3),
}
for name, y in cases.items():
    d = torch.from_numpy(y).cuda()
    for _ in range(3):
        ara.ara_pml_tvar(d, rps)
    pd = torch.zeros(len(rps), dtype=torch.float64, device="cuda")
    td = torch.zeros_like(pd)
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        ara.ara_pml_tvar_device(d, rps, pd, td)
    a.record()
    for _ in range(50):
        ara.ara_pml_tvar_device(d, rps, pd, td)
    b.record()
    torch.cuda.synchronize()
    print(name, "device call (alloc + memset + select) us:", a.elapsed_time(b) * 1e3 / 50, flush=True)
