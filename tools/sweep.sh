#!/bin/bash
# quick config2/config5 timing under env-var variants (no tests)
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/b.json 2> /tmp/b.err
  echo "== $v : $(python -c "import json;d=json.load(open('/tmp/b.json'));print(d['ms_per_step'], d['value'], d['roofline']['kernel'], d['roofline']['frac'])")"
  grep -E "build0|apply0|l=1" /tmp/b.err
  env $v timeout 300 python bench.py --workload config5 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /tmp/b5.json 2> /tmp/b5.err
  echo "   config5: $(python -c "import json;d=json.load(open('/tmp/b5.json'));print(d['ms_per_step'], d['value'], d['roofline']['kernel'], d['roofline']['frac'])")"
  grep -E "build0|apply0|l=1" /tmp/b5.err
done
