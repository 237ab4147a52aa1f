#!/bin/bash
# Same-box A/B/C of the presence kernel's per-window L2 prefetch distance on P (run when option 3 meant four
# windows ahead; option d now means d windows ahead).
O=gpurun_out; mkdir -p $O
for r in 1 2; do
  for pf in 0 2 3; do
    timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --prefetch $pf > $O/bench_pfb${pf}_$r.json 2>/dev/null
    python -c "
import json;d=json.loads(open('$O/bench_pfb${pf}_$r.json').read().strip().splitlines()[-1]);print('pf $pf run $r','step',d['ms_per_step'],'kernel',d['kernel_ms_per_step'])"
  done
done
for pf in 0 2 3; do timeout 300 python bench.py --config M --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-cold --prefetch $pf > $O/bench_M_pf$pf.json 2>/dev/null; python -c "
import json;d=json.loads(open('$O/bench_M_pf$pf.json').read().strip().splitlines()[-1]);print('M pf $pf','step',d['ms_per_step'],'kernel',d['kernel_ms_per_step'])"; done
