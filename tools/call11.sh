python tools/ncu_target.py --workload config5 --frames 8 > gpurun_out/plain11.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_apply|k_build" -s 10 -c 10 -o gpurun_out/prof_c5 python tools/ncu_target.py --workload config5 --frames 8 > gpurun_out/ncu11.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu11.log
bash tools/sweep.sh FLLF_BUILD0_CHUNK=4
