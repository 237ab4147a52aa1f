#!/bin/bash
# Iteration: GPU tests, bench (no e2e/cpu), sweep, ncu full of the default kernel.  Usage: gpu_iter.sh TAG [KREGEX]
TAG=${1:-it}; KRE=${2:-ara_presence_kernel}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --sweep > gpurun_out/bench_$TAG.json 2> gpurun_out/sweep_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 1 -c 1 \
  -o gpurun_out/prof_$TAG -f python bench.py --steps 1 --warmup 1 --profile > gpurun_out/ncu_full_$TAG.log 2>&1
