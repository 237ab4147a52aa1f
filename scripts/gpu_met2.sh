#!/bin/bash
TAG=${1:-met}
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -k "metric or fullsize or plan or dist" > $O/pytest_met_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_met_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-cold > $O/bench_P_$TAG.json 2> $O/bench_P_$TAG.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('$O/bench_P_$TAG.json').read().strip().splitlines()[-1]);print('step',d['ms_per_step'],'kernel',d['kernel_ms_per_step'],'metrics',d['gather_metrics_ms_per_step'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:metrics_select -s 2 -c 1 -o $O/prof_met_$TAG -f python bench.py --steps 2 --warmup 1 --profile > $O/ncu_met_$TAG.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ara_presence_kernel -s 1 -c 1 -o /tmp/prof_P -f python bench.py --steps 1 --warmup 1 --profile > $O/ncu_P_$TAG.log 2>&1; echo "ncu P rc=$?"
ncu -i /tmp/prof_P.ncu-rep --page source --csv --print-source sass > $O/ncu_src_P_$TAG.csv 2>/dev/null
python scripts/ncu_summary.py /tmp/prof_P.ncu-rep > $O/ncu_P_$TAG.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ara_lane_kernel -s 1 -c 1 -o /tmp/prof_X -f python bench.py --config X --steps 1 --warmup 1 --profile > $O/ncu_X_$TAG.log 2>&1; echo "ncu X rc=$?"
ncu -i /tmp/prof_X.ncu-rep --page source --csv --print-source sass > $O/ncu_src_X_$TAG.csv 2>/dev/null
python scripts/ncu_summary.py /tmp/prof_X.ncu-rep > $O/ncu_X_$TAG.txt
