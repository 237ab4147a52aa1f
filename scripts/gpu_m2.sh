#!/bin/bash
TAG=${1:-m}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -q -x > gpurun_out/pytest_stream_$TAG.log 2>&1
timeout 600 python bench.py --config M --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-cold > gpurun_out/bench_M_$TAG.json 2>&1
timeout 300 python bench.py --config X --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-cold --profile > gpurun_out/bench_X_$TAG.json 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --profile --stream 1 > gpurun_out/bench_P_lane_$TAG.json 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --profile > gpurun_out/bench_P_$TAG.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ara_fused_kernel -s 1 -c 1 \
  -o gpurun_out/prof_M_$TAG -f python bench.py --config M --steps 1 --warmup 1 --profile > gpurun_out/ncu_M_$TAG.log 2>&1
