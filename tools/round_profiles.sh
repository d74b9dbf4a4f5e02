#!/bin/bash
# Round artefacts: default bench line (with cpu_baseline), ncu launch list of the
# bench command, ncu --set full of the config-2 kernels.  usage: tools/round_profiles.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/${TAG}_clocks.csv &
SMI=$!
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
kill $SMI
cat gpurun_out/${TAG}_bench.json
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
python tools/ncu_target.py > gpurun_out/${TAG}_plain_t.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_apply|k_build" -s 10 -c 10 \
    -o gpurun_out/${TAG}_full python tools/ncu_target.py > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "full rc=$?"
for w in config5 config4 config3; do
  timeout 300 python bench.py --workload $w --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err
  head -c 300 gpurun_out/${TAG}_bench_$w.json; echo
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_reference.json 2>&1; cat gpurun_out/${TAG}_reference.json
