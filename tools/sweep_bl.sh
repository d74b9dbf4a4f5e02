for v in "FLLF_BL_WARPS=1184" "FLLF_BL_WARPS=600" "FLLF_BL_WARPS=2368" "FLLF_BL_WARPS=4736" "FLLF_BL_RMAX=32 FLLF_BL_WARPS=300" "FLLF_BL_WARPS=9472"; do
  echo "$v: $(env $v python bench.py --workload config2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 >/tmp/j.json | grep -E "build   l=1" | cut -c1-60) $(python -c "import json;print(json.load(open(\"/tmp/j.json\"))[\"ms_per_step\"])")"
  echo "   c5: $(env $v python bench.py --workload config5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 >/tmp/j.json | grep -E "build   l=1" | cut -c1-60) $(python -c "import json;print(json.load(open(\"/tmp/j.json\"))[\"ms_per_step\"])")"
done
