#!/bin/bash
# Same-box A/B of library variants: tools/ab.sh "c2 c5" lib1.so lib2.so ...
# prints one line per (config, lib): value (Mrays/s) and ms/step.
cfgs="$1"; shift
for c in $cfgs; do
  case $c in c3) st="--steps 3 --warmup 3";; c5) st="--steps 3 --warmup 3";; c4) st="--steps 5 --warmup 3";; *) st="--steps 30 --warmup 5";; esac
  for rep in 1 2; do
    for lib in "$@"; do
      out=$(LFP_LIB_PATH=$lib timeout 600 python bench.py --config $c $st --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
      echo "$c rep$rep $(basename $lib) $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],2), d["unit"], round(d["ms_per_step"],3), "frac", round(d["roofline"]["frac"],4))' 2>&1)"
    done
  done
done
