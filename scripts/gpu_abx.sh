#!/bin/bash
# Same-box A/B of build/libA vs build/libB on config X (alternating), then libB's stream tests.
O=gpurun_out; mkdir -p $O
for r in 1 2 3; do
  for v in A B; do
    cp build/lib$v/libara.so paper_1412_4556_b200/libara.so
    X_SWEEP_BASE_ONLY=1 timeout 300 python scripts/probes/x_sweep.py X 2>/dev/null | head -1 | sed "s/^/lib $v run $r /"
  done
done
cp build/libB/libara.so paper_1412_4556_b200/libara.so
timeout 900 python -m pytest tests/test_gpu_stream.py -m gpu -q > $O/pytest_abx.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_abx.log
