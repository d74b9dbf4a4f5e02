#!/bin/bash
# Optional extras: the GPU test suite's timing and a compute-only / end-to-end
# split of the order-sharded config 3 on one GPU.  usage: tools/round_extra.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
start=$(date +%s)
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "gpu tests rc=$? $(( $(date +%s) - start )) s"
tail -3 gpurun_out/${TAG}_gpu_tests.log
