timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/sweep.sh FLLF_BUILD0_CHUNK=4
timeout 300 python bench.py --workload config4 --steps 2 --warmup 1 > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err
timeout 300 python bench.py --workload config3 --steps 3 --warmup 1 > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err; cat gpurun_out/bench_c3.json; tail -3 gpurun_out/bench_c3.err
