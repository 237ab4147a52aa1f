#!/bin/bash
# The whole-trial mask kernel (ARA_OPT_STREAM 11) vs the presence kernel on P, same box, then its tests.
O=gpurun_out; mkdir -p $O
timeout 600 python scripts/probes/p_sweep.py P > $O/p_sweep_wt.txt 2>&1; cat $O/p_sweep_wt.txt
timeout 900 python -m pytest tests/test_gpu_stream.py -m gpu -q > $O/pytest_wt.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_wt.log
timeout 300 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio --clock-control none -k regex:ara_mask_kernel -s 1 -c 1 python bench.py --steps 2 --warmup 1 --profile --stream 11 2>/dev/null | grep -E "inst_executed|duration|issue_active|long_score|ara_mask"
