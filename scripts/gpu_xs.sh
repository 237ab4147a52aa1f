#!/bin/bash
# XS with the compact-row index: parity tests, X bench per XS variant, ncu of the default X kernel
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -q -x -k "exact_scan" > gpurun_out/pytest_xs_${TAG}.log 2>&1
for s in 5 6 7; do timeout 300 python bench.py --config X --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-cold --profile --stream $s > gpurun_out/bench_X_${TAG}_s$s.json 2>&1; done
timeout 300 python bench.py --config X --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-cold --profile > gpurun_out/bench_X_${TAG}.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ara_lane_kernel -s 1 -c 1 \
  -o gpurun_out/prof_X_$TAG -f python bench.py --config X --steps 1 --warmup 1 --profile > gpurun_out/ncu_X_$TAG.log 2>&1
