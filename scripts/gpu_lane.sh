#!/bin/bash
# Round 2: lane-kernel iteration.  Usage: gpu_lane.sh TAG
TAG=${1:-l}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_dist.py -q -x > gpurun_out/pytest_stream_$TAG.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --sweep > gpurun_out/bench_$TAG.json 2> gpurun_out/sweep_$TAG.err
for rm in 16 20 28 32; do timeout 100 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --profile --round-min $rm > gpurun_out/bench_${TAG}_rm$rm.json 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ara_lane_kernel -s 1 -c 1 \
  -o gpurun_out/prof_$TAG -f python bench.py --steps 1 --warmup 1 --profile > gpurun_out/ncu_full_$TAG.log 2>&1
