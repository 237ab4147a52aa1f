#!/bin/bash
# One GPU call: parity tests, H2D probe, ncu launch list + full capture of the ARA kernel, launch-shape sweep.
# Usage (under gpurun): bash scripts/gpu_profile.sh <tag> [config]
TAG=${1:-r1}; CFG=${2:-P}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
timeout 120 python scripts/h2d_probe.py > gpurun_out/h2d_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --config $CFG --steps 3 --warmup 1 --profile > gpurun_out/launches_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ara_layer_kernel -s 1 -c 1 \
  -o gpurun_out/prof_$TAG -f python bench.py --config $CFG --steps 1 --warmup 1 --profile > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --sweep \
  > gpurun_out/sweep_$TAG.json 2> gpurun_out/sweep_$TAG.err
