#!/bin/bash
# Same-box comparison of the fixed-length kernels + lane debug + ncu of the ring kernel.  Usage: gpu_cmp.sh TAG
TAG=${1:-c}
mkdir -p gpurun_out
timeout 300 python scripts/lane_debug.py > gpurun_out/lane_debug_$TAG.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --sweep > gpurun_out/bench_$TAG.json 2> gpurun_out/sweep_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ara_stream_kernel -s 1 -c 1 \
  -o gpurun_out/prof_ring_$TAG -f python bench.py --steps 1 --warmup 1 --profile --stream 4 > gpurun_out/ncu_ring_$TAG.log 2>&1
