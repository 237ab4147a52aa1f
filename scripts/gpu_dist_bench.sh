#!/bin/bash
# The N > 1 bench flow on one GPU: torchrun ranks sharing cuda:0 over gloo (NCCL cannot place two ranks on
# one device); the YLT gather goes through host memory, everything else is the multi-GPU code path.
TAG=${1:-d}
mkdir -p gpurun_out
run() {  # nproc config extra
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29500 + $1)) \
    bench.py --gpus $1 --steps 5 --warmup 3 --dist-backend gloo --no-e2e --no-cold --config $2 $3 > gpurun_out/bench_dist_${2}_n$1_$TAG.json 2> gpurun_out/bench_dist_${2}_n$1_$TAG.err
  echo "n=$1 $2 rc=$?"
}
run 2 P
run 3 P
run 2 M --no-cpu-baseline
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29599 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_dist_ref_$TAG.json 2>&1; echo "ref rc=$?"
