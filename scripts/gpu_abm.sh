#!/bin/bash
# Same-box A/B of two libara.so builds on the captured metric step (scripts/probes/plan_metrics.py), then
# libB's metric tests.
O=gpurun_out; mkdir -p $O
for r in 1 2 3; do
  for v in A B; do
    cp build/lib$v/libara.so paper_1412_4556_b200/libara.so
    timeout 300 python scripts/probes/plan_metrics.py 2>/dev/null | tail -1 | sed "s/^/lib $v run $r: /"
  done
done
cp build/libB/libara.so paper_1412_4556_b200/libara.so
timeout 600 python -m pytest tests -m gpu -q -k "metric" > $O/pytest_abm.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_abm.log
