#!/bin/bash
# One GPU round-trip: parity tests, bench, per-kernel ncu metrics of one filter.
# usage: tools/gpu_check.sh TAG [pytest-args]
TAG=${1:-run}; shift
mkdir -p gpurun_out
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q "$@" 2>&1 | tail -6
fi
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -12 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
python tools/ncu_target.py --workload ${WL:-config2} > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --clock-control none -k regex:"k_apply|k_build" -s 10 -c 10 \
  --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size \
  --csv python tools/ncu_target.py --workload ${WL:-config2} > gpurun_out/ncu_$TAG.csv 2> gpurun_out/ncu_$TAG.err
echo "ncu rc=$?"
