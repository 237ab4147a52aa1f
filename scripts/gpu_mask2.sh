#!/bin/bash
TAG=${1:-k}
mkdir -p gpurun_out
for pf in 0 1; do for pol in 0 1; do
 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --profile --stream 9 --prefetch $pf --l2-policy $pol > gpurun_out/bench_P_${TAG}_pf${pf}_pol${pol}.json 2>&1
done; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cold --profile > gpurun_out/bench_P_${TAG}_pres.json 2>&1
