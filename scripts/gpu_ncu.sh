#!/bin/bash
# ncu full capture of one kernel (source-level) + a quick sweep.  Usage: gpu_ncu.sh TAG KREGEX [CONFIG] [extra bench args]
TAG=${1:-n}; KRE=${2:-ara_stream_kernel}; CFG=${3:-P}; shift 3; EXTRA="$@"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 1 -c 1 \
  -o gpurun_out/prof_$TAG -f python bench.py --config $CFG --steps 1 --warmup 1 --profile $EXTRA > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 400 python bench.py --config $CFG --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --sweep $EXTRA \
  > gpurun_out/sweep_$TAG.json 2> gpurun_out/sweep_$TAG.err
