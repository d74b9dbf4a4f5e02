#!/bin/bash
# Extra round artefacts after tools/round_profiles.sh: ncu --set full of the
# config-5 kernels (4 frames, one filter sequence) and the NEXT-1 / NEXT-3
# bench lines.  usage: tools/round_extra.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
python tools/ncu_target.py --workload config5 --frames 4 > gpurun_out/${TAG}_plain_c5.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_apply|k_build" -s 10 -c 10 \
    -o gpurun_out/${TAG}_c5_full python tools/ncu_target.py --workload config5 --frames 4 > gpurun_out/${TAG}_ncu_c5.log 2>&1
echo "c5 full rc=$?"
for w in bands color; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err
  head -c 300 gpurun_out/${TAG}_bench_$w.json; echo
done
