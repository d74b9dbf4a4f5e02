#!/bin/bash
# A/B of library builds (FLLF_LIB=...; "base" = the in-tree libfllf.so),
# interleaved A B A B ... so clock / power drift hits both alike.
# usage: tools/ab_lib.sh WORKLOAD STEPS REPS lib1 lib2 ...
W=$1; ST=$2; REPS=$3; shift 3
for r in $(seq 1 $REPS); do
  for L in "$@"; do
    if [ "$L" = base ]; then unset FLLF_LIB; else export FLLF_LIB=$PWD/paper_2206_04681_b200/lib/variants/libfllf_$L.so; fi
    timeout 300 python bench.py --workload $W --steps $ST --warmup 5 --no-cpu-baseline --no-e2e > /tmp/ab.json 2> /tmp/ab.err
    echo "== [$L] $W rep $r: $(python -c "import json;d=json.load(open('/tmp/ab.json'));print(d['ms_per_step'],'ms', d['value'],'MP/s', d['clocks']['sm_mhz'])" 2>&1)"
    grep -E "^\[bench\] (build|apply|fuse)" /tmp/ab.err | head -4
  done
done
unset FLLF_LIB
