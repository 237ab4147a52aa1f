"""Small ARA runs for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): configs T and V
through the presence and dense kernels and every fixed-length kernel (lane, ring, lane + exact scan
filter), a wide-row (J = 100) layer over a folded catalogue with and without the exact filter, a fused
multi-layer pass, a captured plan and the metrics, all checked against the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle
from ara_testutil import KERNEL_STREAM, gpu_ylt, select, within_tol
from paper_1412_4556_b200 import ara, synth

bad = 0
for name in ("T", "V"):
    cfg = synth.Config.load(name)
    elts = synth.make_elts(cfg)
    yet = synth.make_yet(cfg)
    if name == "V":  # keep the sanitizer run short
        n = 300
        yet = synth.make_yet(cfg, 0, n)
    want = oracle.ylt_for(cfg, elts, yet)
    ctx = ara.context_for_config(cfg, elts)
    kernels = [(ara.KERNEL_PRESENCE, 0), (ara.KERNEL_DENSE, 0)]
    if name == "T":
        kernels += [(KERNEL_STREAM, 0), (KERNEL_STREAM, 3), (KERNEL_STREAM, 4)]  # lane, ring, lane + XS
    for kern, v in kernels:
        if name == "T":
            y = gpu_ylt(cfg, ctx, yet.event_ids, K=cfg.kmin, kernel=kern, variant=v)
        else:
            y = gpu_ylt(cfg, ctx, yet.event_ids, offsets_np=yet.offsets, kernel=kern, variant=v)
        ok = np.array_equal(y, want) if cfg.regime == "integer" else bool(np.all(within_tol(y, want)))
        print(name, kern, v, ctx.ara_kernel_name(), "ok" if ok else "MISMATCH", flush=True)
        bad += 0 if ok else 1
    rps = synth.return_periods(cfg.num_trials if name == "T" else n)
    import torch
    p_, t_ = ara.ara_pml_tvar(torch.from_numpy(want[0]).cuda(), rps)
    ok = np.array_equal(p_, oracle.pml(want[0], rps))
    print(name, "metrics", "ok" if ok else "MISMATCH", flush=True)
    bad += 0 if ok else 1
# wide rows (J = 100, 416-B rows) over a 3M-event catalogue: folded bitmap, sparse records, filter stage
rng = np.random.default_rng(7)
C, J, N, K = 3_000_000, 100, 64, 1000
elts = []
for j in range(J):
    ids = rng.choice(np.arange(1, C + 1), size=20_000, replace=False).astype(np.uint32)
    elts.append((ids, rng.integers(1, 1 << 20, size=ids.size).astype(np.float32), (float(j % 4) * 1e5, np.inf)))
layer = (list(range(J)), (5000.0, float(1 << 24)), (2e5, 4e7))
yet = rng.integers(1, C + 1, size=N * K).astype(np.uint32)
want = oracle.ylt(C, yet, None, N, K, elts, [layer])
ctx = ara.Context(C, [ara.Elt(i, l, r, lim) for i, l, (r, lim) in elts],
                  [ara.Layer(layer[0], layer[1][0], layer[1][1], layer[2][0], layer[2][1])])
ctx.ara_set_option(ara.ARA_OPT_KERNEL, ara.KERNEL_PRESENCE)
for f in (0, 1):
    ctx.ara_set_option(ara.ARA_OPT_FILTER, f)
    ok = np.array_equal(gpu_ylt(None, ctx, yet, K=K), want)
    print("J=100 filter", f, "ok" if ok else "MISMATCH", flush=True)
    bad += 0 if ok else 1
# fused multi-layer pass and a captured plan (3 layers over distinct ELTs, fixed-length trials)
import torch
C, K, N = 5000, 100, 200
elts = []
for j in range(12):
    ids = rng.choice(np.arange(1, C + 1), size=300, replace=False).astype(np.uint32)
    elts.append((ids, rng.integers(1, 1 << 20, size=ids.size).astype(np.float32), (float(j % 3) * 1e4, np.inf)))
layers = [(list(range(4 * l, 4 * l + 4)), (100.0 * l, 5e6), (1e4 * l, 4e7)) for l in range(3)]
yet = rng.integers(1, C + 1, size=N * K).astype(np.uint32)
want = oracle.ylt(C, yet, None, N, K, elts, layers)
ctx = ara.Context(C, [ara.Elt(i, l, r, lim) for i, l, (r, lim) in elts],
                  [ara.Layer(l[0], l[1][0], l[1][1], l[2][0], l[2][1]) for l in layers])
ctx.ara_set_option(ara.ARA_OPT_FUSED, 1)
ok = np.array_equal(gpu_ylt(None, ctx, yet, K=K, num_trials=N, num_layers=3), want)
print("fused", ctx.ara_kernel_name(), "ok" if ok else "MISMATCH", flush=True)
bad += 0 if ok else 1
ctx.ara_set_option(ara.ARA_OPT_FUSED, 0)
ids = torch.from_numpy(yet.view(np.int32)).cuda()
y = torch.zeros((3, N), dtype=torch.float64, device="cuda")
rps = synth.return_periods(N)
pm = torch.zeros((3, len(rps)), dtype=torch.float64, device="cuda")
tv = torch.zeros((3, len(rps)), dtype=torch.float64, device="cuda")
plan = ctx.ara_plan_create(ids, y, rps, pm, tv, events_per_trial=K, num_trials=N)
plan.launch()
torch.cuda.synchronize()
ok = np.array_equal(y.cpu().numpy(), want) and np.array_equal(pm[0].cpu().numpy(), oracle.pml(want[0], rps))
print("plan", "ok" if ok else "MISMATCH", flush=True)
bad += 0 if ok else 1
plan.close()
sys.exit(1 if bad else 0)
