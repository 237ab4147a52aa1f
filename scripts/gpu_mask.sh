#!/bin/bash
TAG=${1:-k}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -q -x -k "mask" > gpurun_out/pytest_mask_$TAG.log 2>&1
for s in 9 10 0; do timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --profile --stream $s > gpurun_out/bench_P_${TAG}_s$s.json 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ara_mask_kernel -s 1 -c 1 \
  -o gpurun_out/prof_mask_$TAG -f python bench.py --steps 1 --warmup 1 --profile --stream 9 > gpurun_out/ncu_mask_$TAG.log 2>&1
