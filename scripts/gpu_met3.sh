#!/bin/bash
TAG=${1:-met}
O=gpurun_out; mkdir -p $O
python scripts/probes/metrics_trace.py > $O/mtrace_$TAG.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "metric or fullsize or plan or dist" > $O/pytest_met_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_met_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-cold > $O/bench_P_$TAG.json 2> $O/bench_P_$TAG.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('$O/bench_P_$TAG.json').read().strip().splitlines()[-1]);print('step',d['ms_per_step'],'kernel',d['kernel_ms_per_step'],'metrics',d['gather_metrics_ms_per_step'])"
