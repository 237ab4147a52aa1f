#!/bin/bash
# Round-2 artifacts in one GPU call (copied into profiles/ afterwards): GPU tests, compute-sanitizer
# (memcheck, racecheck, synccheck, initcheck), the default bench line + reference arm, every config's
# bench line, the ncu launch list of the default bench command, ncu --set full captures (P presence,
# X lane+XS, M fused) summarised, and the Section IV.B study with per-layout ncu counters.
TAG=${1:-r2}
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
for T in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $T --error-exitcode 9 python scripts/sanitize_run.py > $O/sanitize_${T}_$TAG.log 2>&1
  echo "sanitizer $T rc=$?" | tee -a $O/sanitize_summary_$TAG.txt
done
timeout 900 python bench.py > $O/bench_P_$TAG.json 2> $O/bench_P_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_P_$TAG.json 2> $O/bench_ref_P_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_P_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --profile > $O/launches_bench_$TAG.log 2>&1
python scripts/launch_summary.py $O/launches_P_$TAG.csv > $O/launches_P_$TAG.txt
prof() {  # config kernel-regex extra-args
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 \
    -o /tmp/prof_$1_$TAG -f python bench.py --config $1 --steps 1 --warmup 1 --profile $3 > $O/ncu_full_$1_$TAG.log 2>&1
  python scripts/ncu_summary.py /tmp/prof_$1_$TAG.ncu-rep --json $O/ncu_$1_$TAG.json --config $1 --variant "$4" > $O/ncu_$1_$TAG.txt
  ncu -i /tmp/prof_$1_$TAG.ncu-rep --page source --csv --print-source sass > $O/ncu_src_$1_$TAG.csv 2>/dev/null
}
prof P ara_presence_kernel "" "ara_presence_kernel<V=8,NV=2,G=1,NW=32>"
prof X ara_lane_kernel "" "ara_lane_kernel<NW=24,XS>"
for C in M X PI V; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 > $O/bench_${C}_$TAG.json 2> $O/bench_${C}_$TAG.err
done
timeout 900 python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-cold --profile --study \
  > $O/bench_study_$TAG.json 2> $O/study_$TAG.err
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum \
  --clock-control none --csv --log-file $O/study_ncu_$TAG.csv -k regex:study_kernel \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-cold --profile --study > $O/study_ncu_$TAG.log 2>&1
echo done
