#!/bin/bash
# Same-box A/B of two builds of libara.so (build/libA, build/libB), alternating, P and M.
O=gpurun_out; mkdir -p $O
for r in 1 2 3; do
  for v in A B; do
    cp build/lib$v/libara.so paper_1412_4556_b200/libara.so
    timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --no-cold > $O/ab_${v}_$r.json 2>/dev/null
    python -c "
import json;d=json.loads(open('$O/ab_${v}_$r.json').read().strip().splitlines()[-1]);print('lib $v run $r','step',d['ms_per_step'],'kernel',d['kernel_ms_per_step'])"
  done
done
for v in A B; do
  cp build/lib$v/libara.so paper_1412_4556_b200/libara.so
  timeout 300 python bench.py --config M --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-cold > $O/ab_M_$v.json 2>/dev/null
  python -c "
import json;d=json.loads(open('$O/ab_M_$v.json').read().strip().splitlines()[-1]);print('M lib $v','step',d['ms_per_step'],'kernel',d['kernel_ms_per_step'])"
done
cp build/libB/libara.so paper_1412_4556_b200/libara.so
