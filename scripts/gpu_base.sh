#!/bin/bash
# Session baseline: GPU tests, the default bench line, X and M bench lines.
TAG=${1:-base}
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_P_$TAG.json 2> $O/bench_P_$TAG.err; echo "bench P rc=$?"
timeout 600 python bench.py --config X --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-cold > $O/bench_X_$TAG.json 2> $O/bench_X_$TAG.err; echo "bench X rc=$?"
