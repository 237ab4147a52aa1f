"""Small ARA runs for compute-sanitizer (memcheck / racecheck / synccheck): configs T and V through the
presence and dense kernels, checked against the oracle."""
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
sys.exit(1 if bad else 0)
