#!/bin/bash
# Configs M and X with both kernels + P metrics launch list.  Usage: gpu_configs.sh TAG
TAG=${1:-cfg}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "metrics or sharded or extended" > gpurun_out/pytest_gpu_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 1 --profile > /dev/null 2>&1
for K in presence dense; do
  timeout 900 python bench.py --config M --steps 5 --warmup 3 --no-e2e --no-cold --kernel $K > gpurun_out/bench_M_${K}_$TAG.json 2> gpurun_out/bench_M_${K}_$TAG.err
  timeout 1200 python bench.py --config X --steps 5 --warmup 3 --no-e2e --no-cold --kernel $K --cpu-sample 8192 > gpurun_out/bench_X_${K}_$TAG.json 2> gpurun_out/bench_X_${K}_$TAG.err
done
