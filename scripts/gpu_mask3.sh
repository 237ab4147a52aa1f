#!/bin/bash
# mask kernel (stream 9: NW=32, 10: NW=24) against the presence kernel on the same box
TAG=${1:-k}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py -q -x -k mask > gpurun_out/mask_tests_${TAG}.log 2>&1
for rep in 0 1; do
for st in 9 10; do
 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --profile --stream $st --prefetch 0 > gpurun_out/bench_P_${TAG}_s${st}_r${rep}.json 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --profile > gpurun_out/bench_P_${TAG}_pres_r${rep}.json 2>&1
done
