#!/bin/bash
# Same-box A/B of build/libA vs build/libB (alternating, P and M), then libB's parity tests.
O=gpurun_out; mkdir -p $O
bash scripts/gpu_ab.sh
cp build/libB/libara.so paper_1412_4556_b200/libara.so
timeout 900 python -m pytest tests -m gpu -q -k "stream or parity or fullsize" > $O/pytest_ab2.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_ab2.log
timeout 300 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:ara_presence_kernel -s 1 -c 1 python bench.py --steps 2 --warmup 1 --profile 2>/dev/null | grep -E "inst_executed|duration|ara_presence"
