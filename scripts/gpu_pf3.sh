#!/bin/bash
# Same-box A/B: presence kernel without / with the per-window L2 prefetch (constant-offset form), on P and M,
# and the instruction count of each under ncu.
O=gpurun_out; mkdir -p $O
for r in 1 2; do
  for pf in 0 2; do
    timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --prefetch $pf > $O/bench_pfc${pf}_$r.json 2>/dev/null
    python -c "
import json;d=json.loads(open('$O/bench_pfc${pf}_$r.json').read().strip().splitlines()[-1]);print('pf $pf run $r','step',d['ms_per_step'],'kernel',d['kernel_ms_per_step'])"
  done
done
for pf in 0 2; do timeout 300 python bench.py --config M --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-cold --prefetch $pf > $O/bench_M_pfc$pf.json 2>/dev/null; python -c "
import json;d=json.loads(open('$O/bench_M_pfc$pf.json').read().strip().splitlines()[-1]);print('M pf $pf','step',d['ms_per_step'],'kernel',d['kernel_ms_per_step'])"; done
for pf in 0 2; do timeout 300 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio --clock-control none -k regex:ara_presence_kernel -s 1 -c 1 python bench.py --steps 2 --warmup 1 --profile --prefetch $pf 2>/dev/null | grep -E "inst_executed|duration|long_score" | sed "s/^/pf $pf /"; done
