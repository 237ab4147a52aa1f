#!/bin/bash
TAG=${1:-x}
mkdir -p gpurun_out
for s in 5 6 7; do timeout 300 python bench.py --config X --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-cold --profile --stream $s > gpurun_out/bench_X_${TAG}_s$s.json 2>&1; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --profile > gpurun_out/bench_P_${TAG}.json 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --profile --eager > gpurun_out/bench_P_${TAG}_eager.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:metrics_fused -s 2 -c 1 \
  -o gpurun_out/prof_metrics_$TAG -f python bench.py --steps 2 --warmup 1 --profile > gpurun_out/ncu_metrics_$TAG.log 2>&1
