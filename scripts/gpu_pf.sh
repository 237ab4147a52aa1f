#!/bin/bash
# Same-box A/B of the presence kernel's per-window L2 prefetch (ARA_OPT_PREFETCH 2) on P.
O=gpurun_out; mkdir -p $O
for r in 1 2; do
  for pf in -1 2; do
    timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --prefetch $pf > $O/bench_pf${pf}_$r.json 2>/dev/null
    python -c "
import json;d=json.loads(open('$O/bench_pf${pf}_$r.json').read().strip().splitlines()[-1]);print('pf $pf run $r','step',d['ms_per_step'],'kernel',d['kernel_ms_per_step'])"
  done
done
timeout 300 python -m pytest tests -m gpu -q -k "determinism or prefetch" > $O/pytest_pf.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_pf.log
