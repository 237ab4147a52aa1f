#!/bin/bash
TAG=${1:-t2}
O=gpurun_out; mkdir -p $O
./scripts/probes/barrier_probe > $O/barrier_probe.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -5 $O/pytest_gpu_$TAG.log
