#!/bin/bash
# Round-2 final artifacts in one GPU call (compute-sanitizer is closed on the pool; the full-oracle
# cpu_baseline line is r2b): GPU tests, the default bench line, the reference arm, the launch list of the default bench command, ncu --set full captures of the P presence
# kernel, the X lane+XS kernel and metrics_select (summaries + SASS source CSVs), every config's bench line.
TAG=${1:-r2c}
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu_$TAG.log
timeout 900 python bench.py > $O/bench_P_$TAG.json 2> $O/bench_P_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_P_$TAG.json 2> $O/bench_ref_P_$TAG.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_P_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --profile > $O/launches_bench_$TAG.log 2>&1
python scripts/launch_summary.py $O/launches_P_$TAG.csv > $O/launches_P_$TAG.txt
prof() {  # name config kernel-regex skip extra-args
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 \
    -o /tmp/prof_$1_$TAG -f python bench.py --config $2 --steps 2 --warmup 1 --profile > $O/ncu_full_$1_$TAG.log 2>&1
  echo "ncu $1 rc=$?"
  python scripts/ncu_summary.py /tmp/prof_$1_$TAG.ncu-rep > $O/ncu_$1_$TAG.txt
  ncu -i /tmp/prof_$1_$TAG.ncu-rep --page source --csv --print-source sass > $O/ncu_src_$1_$TAG.csv 2>/dev/null
}
prof P P ara_presence_kernel 1
prof X X ara_lane_kernel 1
prof metrics P metrics_select 2
for C in M X PI V; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 > $O/bench_${C}_$TAG.json 2> $O/bench_${C}_$TAG.err
  echo "bench $C rc=$?"
done
echo done
