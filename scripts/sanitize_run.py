"""Small ARA runs for compute-sanitizer (memcheck / racecheck / synccheck): configs T and V through the
presence and dense kernels, and a wide-row (J = 100) layer over a folded catalogue through the record
presence kernel with and without its exact filter stage, checked against the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle
from ara_testutil import gpu_ylt, within_tol
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
    for kern in (ara.KERNEL_PRESENCE, ara.KERNEL_DENSE):
        if name == "T":
            y = gpu_ylt(cfg, ctx, yet.event_ids, K=cfg.kmin, kernel=kern, variant=0)
        else:
            y = gpu_ylt(cfg, ctx, yet.event_ids, offsets_np=yet.offsets, kernel=kern, variant=0)
        ok = np.array_equal(y, want) if cfg.regime == "integer" else bool(np.all(within_tol(y, want)))
        print(name, kern, "ok" if ok else "MISMATCH", flush=True)
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
sys.exit(1 if bad else 0)
