#!/bin/bash
# tests + e2e probe + bench (presence default) + sweeps of both kernels
TAG=${1:-r1b}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
timeout 300 python scripts/e2e_probe.py > gpurun_out/e2e_probe_$TAG.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --sweep \
  > gpurun_out/sweep_$TAG.json 2> gpurun_out/sweep_$TAG.err
