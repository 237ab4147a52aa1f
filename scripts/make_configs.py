"""Write configs/{T,P,P2,M,X,V}.json: workload shapes of BASELINE.json plus frozen financial terms.

Shapes: BASELINE.json "configs" (tiny / paper-shaped / sharded / multi-layer / stress) and SURVEY.md
8(d) (V, variable trial lengths k in [800, 1500]).  Terms (SURVEY.md 8(d) "Terms"):
    mu  = closed-form mean of the integer-regime loss
    FT1_g = (round(mu/8 * (g mod 4)),  +inf if g odd else round(8 mu))
    FT2   = (round(mu/4), round(4 mu))                     (per layer l of M: scaled by 1 + l/8, 1 + l/4)
    FT3   = (q30(S_n), q80(S_n) - q30(S_n))  with S_n the pre-FT3 trial sums of the first pilot
            trials, computed by the ORACLE (this script calls only oracle/ and the shared generator).
Real-regime terms carry two decimal digits.  Run once; the JSON files are committed.
"""
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1412_4556_b200 import synth  # noqa: E402

MU = synth.loss_mean_integer()


def r2(x, regime):
    return round(x, 2) if regime == "real" else float(round(x))


def ft1(g, regime):
    frac = 1.0 + (0.00137 * (g % 7) if regime == "real" else 0.0)
    ret = r2(MU / 8 * (g % 4) * frac, regime)
    lim = math.inf if g % 2 else r2(8 * MU * frac, regime)
    return synth.Terms(ret, lim)


def base_config(name, N, kmin, kmax, C, J_per_layer, n_layers, entries, regime, desc, distinct=True):
    n_elts = J_per_layer * n_layers if distinct else J_per_layer
    elt_terms = [ft1(g, regime) for g in range(n_elts)]
    layers = []
    for l in range(n_layers):
        elts = list(range(l * J_per_layer, (l + 1) * J_per_layer)) if distinct else list(range(J_per_layer))
        occ = synth.Terms(r2(MU / 4 * (1 + l / 8) * (1.00211 if regime == "real" else 1), regime),
                          r2(4 * MU * (1 + l / 4) * (1.00117 if regime == "real" else 1), regime))
        layers.append(synth.LayerSpec(elts, occ, synth.Terms(0.0, math.inf)))
    return synth.Config(name=name, num_trials=N, kmin=kmin, kmax=kmax, catalog_size=C, entries_per_elt=entries,
                        elt_terms=elt_terms, layers=layers, regime=regime, description=desc)


def set_ft3(cfg, pilot_trials):
    t0 = time.time()
    elts = synth.make_elts(cfg)
    yet = synth.make_yet(cfg, 0, min(cfg.num_trials, pilot_trials))
    S = oracle.ylt_for(cfg, elts, yet)  # FT3 is identity here -> pre-FT3 sums S_n
    for l, layer in enumerate(cfg.layers):
        s = np.sort(S[l])
        q30 = float(s[int(0.3 * (s.size - 1))])
        q80 = float(s[int(0.8 * (s.size - 1))])
        lim = q80 - q30 if q80 > q30 else MU
        layer.agg = synth.Terms(r2(q30, cfg.regime), r2(lim, cfg.regime))
    print(f"  {cfg.name}: pilot {yet.num_trials} trials in {time.time() - t0:.1f}s", flush=True)
    return cfg


def main():
    out = os.path.join(ROOT, "configs")
    os.makedirs(out, exist_ok=True)
    cfgs = [
        (base_config("T", 1000, 100, 100, 10_000, 2, 1, 1000, "integer",
                     "tiny ARA: 1,000 trials x 100 events, 1 layer x 2 ELTs of 1,000 entries, 10,000-event catalog "
                     "(BASELINE.json configs[0]); integer regime (bitwise parity)"), 1000),
        (base_config("P", 1_000_000, 1000, 1000, 2_000_000, 16, 1, 10_000, "real",
                     "paper-shaped ARA: 1M trials x 1,000 events, 1 layer x 16 ELTs x 10,000 entries, 2M-event "
                     "catalog (BASELINE.json configs[1]; PAPER.md:230)"), 10_000),
        (base_config("PI", 1_000_000, 1000, 1000, 2_000_000, 16, 1, 10_000, "integer",
                     "paper-shaped ARA, integer regime (bitwise parity at full size)"), 10_000),
        (base_config("M", 1_000_000, 1000, 1000, 2_000_000, 16, 8, 10_000, "real",
                     "multi-layer ARA: 8 layers sharing one 1M-trial YET, 16 distinct ELTs each, distinct "
                     "occurrence/aggregate terms per layer (BASELINE.json configs[3]; reading c20)"), 10_000),
        (base_config("X", 8_000_000, 1000, 1000, 10_000_000, 100, 1, 10_000, "real",
                     "stress ARA: 8M trials x 1,000 events (32 GB YET), 100 ELTs of 10,000 entries over a "
                     "10M-event catalog (BASELINE.json configs[4]; reading c21)"), 2000),
        (base_config("V", 10_000, 800, 1500, 2_000_000, 16, 1, 10_000, "real",
                     "variable-length trials k ~ U[800,1500] (PAPER.md:57), correctness only"), 10_000),
    ]
    only = set(sys.argv[1:])
    for cfg, pilot in cfgs:
        if only and cfg.name not in only:
            continue
        set_ft3(cfg, pilot)
        with open(os.path.join(out, f"{cfg.name}.json"), "w") as f:
            json.dump(cfg.to_json(), f, indent=1)


if __name__ == "__main__":
    main()
