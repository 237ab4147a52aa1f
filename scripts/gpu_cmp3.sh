#!/bin/bash
TAG=${1:-c}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_$TAG.log 2>&1
for s in 5 6; do timeout 300 python bench.py --config X --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-cold --profile --stream $s > gpurun_out/bench_X_${TAG}_s$s.json 2>&1; done
timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --sweep > gpurun_out/bench_P_$TAG.json 2> gpurun_out/sweep_$TAG.err
