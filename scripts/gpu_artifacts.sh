#!/bin/bash
# One GPU call that regenerates the judged artifacts for a round (copied into profiles/ afterwards):
# GPU tests, the default bench line (+ reference arm), the ncu launch list of the bench command, one
# ncu --set full capture of the presence kernel, the other configs, and the Section IV.B study.
# Usage (under gpurun): bash scripts/gpu_artifacts.sh <tag>
TAG=${1:-art}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py > $O/bench_P_$TAG.json 2> $O/bench_P_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_P_$TAG.json 2> $O/bench_ref_P_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_P_$TAG.csv \
  python bench.py --steps 3 --warmup 1 --profile > $O/launches_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ara_presence_kernel -s 1 -c 1 \
  -o $O/prof_P_$TAG -f python bench.py --steps 1 --warmup 1 --profile > $O/ncu_full_P_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ara_layer_kernel -s 1 -c 1 \
  -o $O/prof_dense_P_$TAG -f python bench.py --steps 1 --warmup 1 --profile --kernel dense > $O/ncu_dense_P_$TAG.log 2>&1
for C in M X PI V; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 > $O/bench_${C}_$TAG.json 2> $O/bench_${C}_$TAG.err
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --study > $O/study_P_$TAG.log 2>&1
echo done
