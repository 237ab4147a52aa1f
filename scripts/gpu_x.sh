#!/bin/bash
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_dist.py -q -x > gpurun_out/pytest_stream_$TAG.log 2>&1
timeout 600 python bench.py --config X --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-cold > gpurun_out/bench_X_$TAG.json 2> gpurun_out/bench_X_$TAG.err
for s in 0 1 5; do timeout 300 python bench.py --config X --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-cold --profile --stream $s --filter 0 > gpurun_out/bench_X_${TAG}_s$s.json 2>&1; done
timeout 900 ncu --set full --clock-control none -k regex:ara_lane_kernel -s 1 -c 1 \
  -o gpurun_out/prof_X_$TAG -f python bench.py --config X --steps 1 --warmup 1 --profile > gpurun_out/ncu_X_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
