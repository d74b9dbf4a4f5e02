#!/bin/bash
# A/B timing of env-var variants on one workload (default config2; no tests, no ncu).
# usage: WL=config2 tools/ab1.sh "VAR=a" "VAR=b" ...
w=${WL:-config2}
for v in "$@"; do
  st=30; [ $w = config5 ] && st=3
  env $v timeout 300 python bench.py --workload $w --steps $st --warmup 3 --no-cpu-baseline --no-e2e > /tmp/ab.json 2> /tmp/ab.err
  echo "== [$v] $w: $(python -c "import json;d=json.load(open('/tmp/ab.json'));print(d['ms_per_step'],'ms', d['value'],'MP/s', d['roofline']['kernel'], d['roofline']['frac'])" 2>&1)"
  grep -E "^\[bench\] (build|apply|coll)" /tmp/ab.err | head -12
done
