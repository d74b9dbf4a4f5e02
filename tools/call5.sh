python tools/ncu_target.py > gpurun_out/plain5.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_apply|k_build" -s 10 -c 10 -o gpurun_out/prof_v3 python tools/ncu_target.py > gpurun_out/ncu5.log 2>&1
echo "ncu rc=$?"
timeout 600 python bench.py --workload config5 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_v3.json 2> gpurun_out/bench_c5_v3.err
tail -12 gpurun_out/bench_c5_v3.err; cat gpurun_out/bench_c5_v3.json
