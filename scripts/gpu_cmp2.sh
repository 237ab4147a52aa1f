#!/bin/bash
TAG=${1:-c}
mkdir -p gpurun_out
timeout 300 python scripts/lane_debug.py > gpurun_out/lane_debug_$TAG.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --sweep > gpurun_out/bench_$TAG.json 2> gpurun_out/sweep_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ara_presence_kernel -s 1 -c 1 \
  -o gpurun_out/prof_pres_$TAG -f python bench.py --steps 1 --warmup 1 --profile --stream 0 > gpurun_out/ncu_pres_$TAG.log 2>&1
