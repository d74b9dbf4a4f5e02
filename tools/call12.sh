timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/sweep.sh FLLF_BUILD0_CHUNK=4
python tools/sanitize_target.py > gpurun_out/san_plain.log 2>&1 && timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_target.py > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/memcheck.log
