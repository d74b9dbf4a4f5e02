#!/bin/bash
# config2-only A/B of env-var variants: bench line + per-kernel times, then the graph level sweep.
for v in "$@"; do
  env $v timeout 300 python bench.py --workload config2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > /tmp/ab.json 2> /tmp/ab.err
  echo "== [$v] config2: $(python -c "import json;d=json.load(open('/tmp/ab.json'));print(d['ms_per_step'],'ms', d['value'],'MP/s', d['roofline']['kernel'], d['roofline']['frac'])" 2>&1)"
  grep -E "^\[bench\] (build|apply)" /tmp/ab.err | head -4
done
