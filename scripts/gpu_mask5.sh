#!/bin/bash
# mask kernel A/B: stream 9 (original), 10 (PFD 4), 11 (unconditional loads), 12 (staging fast path),
# 13 (both), 14 (unconditional loads + PFD 4); presence kernel beside
TAG=${1:-k}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py -q -x -k mask > gpurun_out/mask_tests_${TAG}.log 2>&1
for st in 9 10 11 12 13 14; do
 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --profile --stream $st --prefetch 0 > gpurun_out/bench_P_${TAG}_s${st}.json 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --profile > gpurun_out/bench_P_${TAG}_pres.json 2>&1
