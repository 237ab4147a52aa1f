#!/bin/bash
# Round 2: stream-kernel iteration.  Usage: gpu_stream.sh TAG
TAG=${1:-s}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py -q -x > gpurun_out/pytest_stream_$TAG.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --sweep > gpurun_out/bench_$TAG.json 2> gpurun_out/sweep_$TAG.err
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
