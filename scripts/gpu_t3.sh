#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -k "metric" > $O/pytest_met_t3.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_met_t3.log
timeout 600 python bench.py --config X --steps 10 --warmup 3 > $O/bench_X_t3.json 2> $O/bench_X_t3.err; echo "bench X rc=$?"
