#!/bin/bash
# One GPU call's round artefacts (round 2 layout):
#   default bench line (BASELINE configs[4], with cpu_baseline / e2e) + clocks,
#   config2 / config3 / config4 / bands / color bench lines, the reference arm,
#   the ncu launch list of the default bench command, ncu --set full of one
#   filter sequence at config 5 (8 frames, the 64-frame bench's design choice)
#   and at config 2.
# usage: tools/round_profiles.sh TAG     (then: python tools/collect_profiles.py TAG)
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/${TAG}_clocks.csv &
SMI=$!
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
kill $SMI
cat gpurun_out/${TAG}_bench.json
for w in config2 config3 config4 bands color; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err
  head -c 300 gpurun_out/${TAG}_bench_$w.json; echo
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${TAG}_reference.json 2>&1; tail -c 400 gpurun_out/${TAG}_reference.json
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
python tools/ncu_target.py --workload config5 --frames 8 --iters 1 > gpurun_out/${TAG}_plain_c5.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_apply|k_build|k_fuse|k_collapse" -c 10 \
    -o gpurun_out/${TAG}_c5_full -f python tools/ncu_target.py --workload config5 --frames 8 --iters 1 > gpurun_out/${TAG}_ncu_c5.log 2>&1
echo "c5 full rc=$?"
python tools/ncu_target.py --workload config2 --iters 1 > gpurun_out/${TAG}_plain_c2.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_apply|k_build|k_fuse|k_collapse" -c 10 \
    -o gpurun_out/${TAG}_c2_full -f python tools/ncu_target.py --workload config2 --iters 1 > gpurun_out/${TAG}_ncu_c2.log 2>&1
echo "c2 full rc=$?"
# keep the raw metric pages only (gpurun copies back <= 64 MiB)
for r in c5_full c2_full; do
  if [ -f gpurun_out/${TAG}_$r.ncu-rep ]; then
    ncu -i gpurun_out/${TAG}_$r.ncu-rep --page raw --csv > gpurun_out/${TAG}_${r}_raw.csv 2>/dev/null && rm -f gpurun_out/${TAG}_$r.ncu-rep
  fi
done
