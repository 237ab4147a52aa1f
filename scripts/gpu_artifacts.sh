#!/bin/bash
# One GPU call that regenerates the judged artifacts for a round (copied into profiles/ afterwards):
# GPU tests, compute-sanitizer, the default bench line (+ reference arm), the ncu launch list of the bench
# command, ncu --set full captures of the presence kernel on P and X (summaries + SASS source CSV; the
# .ncu-rep files stay in /tmp: they exceed gpurun's copy-back limit), and the other configs.
# Usage (under gpurun): bash scripts/gpu_artifacts.sh <tag>
TAG=${1:-art}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
for T in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $T --error-exitcode 9 python scripts/sanitize_run.py > $O/sanitize_${T}_$TAG.log 2>&1
  echo "sanitizer $T rc=$?" | tee -a $O/sanitize_summary_$TAG.txt
done
timeout 600 python bench.py > $O/bench_P_$TAG.json 2> $O/bench_P_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_P_$TAG.json 2> $O/bench_ref_P_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_P_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --profile > $O/launches_bench_$TAG.log 2>&1
python scripts/launch_summary.py $O/launches_P_$TAG.csv > $O/launches_P_$TAG.txt
for C in P X; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ara_presence_kernel -s 1 -c 1 \
    -o /tmp/prof_${C}_$TAG -f python bench.py --config $C --steps 1 --warmup 1 --profile > $O/ncu_full_${C}_$TAG.log 2>&1
  V=$(python -c "import json;print(json.load(open('$O/bench_P_$TAG.json'))['config']['kernel'])" 2>/dev/null)
  [ $C = X ] && V="ara_presence_kernel<V=8,NV=13,G=1,NW=32>"
  python scripts/ncu_summary.py /tmp/prof_${C}_$TAG.ncu-rep --json $O/ncu_${C}_$TAG.json --config $C --variant "$V" > $O/ncu_${C}_$TAG.txt
  ncu -i /tmp/prof_${C}_$TAG.ncu-rep --page source --csv --print-source sass > $O/ncu_src_${C}_$TAG.csv 2>/dev/null
done
for C in M X PI V; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 > $O/bench_${C}_$TAG.json 2> $O/bench_${C}_$TAG.err
done
echo done
