#!/bin/bash
# mask kernel: stream 9 (no window prefetch) / 10 (per-lane L2 prefetch 4 windows ahead) x YET L2 policy
# (0: evict_last, 1: evict_normal), against the presence kernel on the same box
TAG=${1:-k}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py -q -x -k mask > gpurun_out/mask_tests_${TAG}.log 2>&1
for st in 9 10; do for pol in 0 1; do
 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --profile --stream $st --prefetch 0 --l2-policy $pol > gpurun_out/bench_P_${TAG}_s${st}_pol${pol}.json 2>&1
done; done
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --profile > gpurun_out/bench_P_${TAG}_pres.json 2>&1
