#!/bin/bash
# After the presence kernel's per-window L2 prefetch became the default: GPU suite, P/PI/M/V bench lines,
# launch list and an ncu capture of the presence kernel.
TAG=${1:-r2d}
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu_$TAG.log
timeout 900 python bench.py > $O/bench_P_$TAG.json 2> $O/bench_P_$TAG.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_P_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --profile > $O/launches_bench_$TAG.log 2>&1
python scripts/launch_summary.py $O/launches_P_$TAG.csv > $O/launches_P_$TAG.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ara_presence_kernel -s 1 -c 1 \
  -o /tmp/prof_P_$TAG -f python bench.py --config P --steps 2 --warmup 1 --profile > $O/ncu_full_P_$TAG.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py /tmp/prof_P_$TAG.ncu-rep > $O/ncu_P_$TAG.txt
ncu -i /tmp/prof_P_$TAG.ncu-rep --page source --csv --print-source sass > $O/ncu_src_P_$TAG.csv 2>/dev/null
for C in PI M V; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 > $O/bench_${C}_$TAG.json 2> $O/bench_${C}_$TAG.err; echo "bench $C rc=$?"
done
