timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/ncu_target.py > gpurun_out/plain9.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_apply|k_build" -s 10 -c 10 -o gpurun_out/prof_v6 python tools/ncu_target.py > gpurun_out/ncu9.log 2>&1
echo "ncu rc=$?"
bash tools/sweep.sh FLLF_BUILD0_CHUNK=4 FLLF_BUILD0_CHUNK=8
