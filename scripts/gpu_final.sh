#!/bin/bash
# Final check of the committed tree: the GPU suite, smoke(), the default bench line.
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_final.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_final.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_P_final.json 2> $O/bench_P_final.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('$O/bench_P_final.json').read().strip().splitlines()[-1]);print('step',d['ms_per_step'],'kernel',d['kernel_ms_per_step'],'metrics',d['gather_metrics_ms_per_step'],'e2e',d['e2e']['value'],'frac',d['roofline']['frac'])"
