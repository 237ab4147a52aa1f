"""Debug: fused vs layer-outer on config M at full size; oracle on the differing trials."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_1412_4556_b200 import ara, synth
cfg = synth.Config.load("M")
elts = synth.make_elts(cfg)
N, K, L = cfg.num_trials, cfg.kmin, len(cfg.layers)
dev = torch.device("cuda:0")
ids = torch.empty(N * K, dtype=torch.int32, device=dev)
synth.yet_ids_device(ids.data_ptr(), cfg.seed, cfg.catalog_size, 0, N * K, torch.cuda.current_stream().cuda_stream)
ctx = ara.context_for_config(cfg, elts)
y = torch.zeros((L, N), dtype=torch.float64, device=dev)
ctx.ara_run(ids, y, events_per_trial=K, num_trials=N); ctx.ara_check()
print("fused kernel:", ctx.ara_kernel_name())
fused = y.cpu().numpy()
ctx.ara_set_option(ara.ARA_OPT_FUSED, 0)
y.zero_()
ctx.ara_run(ids, y, events_per_trial=K, num_trials=N); ctx.ara_check()
outer = y.cpu().numpy()
d = np.abs(fused - outer) > np.maximum(1e-12 * np.abs(outer), 1e-6)
print("differing elements:", int(d.sum()), "per layer:", d.sum(axis=1).tolist())
bad = np.argwhere(d)[:10]
print("first:", bad.tolist())
trials = np.unique(bad[:, 1])[:10]
if len(trials):
    want = oracle.ylt_for(cfg, elts, synth.make_yet_trials(cfg, trials))
    for i, t in enumerate(trials):
        print(t, "fused", fused[:, t].tolist(), "\n   outer", outer[:, t].tolist(), "\n   oracle", want[:, i].tolist())
