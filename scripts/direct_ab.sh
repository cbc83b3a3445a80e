#!/bin/bash
# The posterior-free resident kernel on the C5 n=1008 bench workload (A/B of builds via LDPCB_LIBRARY).
mkdir -p gpurun_out
B="python bench.py --workload c5_n1008 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
run() { # label, env...
  local label=$1; shift
  env "$@" $B 2> gpurun_out/ab_err.log | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l)
        print('$label', 'ms', round(d['ms_per_step'], 3), 'frac', round(d['roofline']['frac'], 4), 'FER', d['counters']['frame_errors'] / d['counters']['frames'], 'BE', d['counters']['bit_errors'], d['config']['plan'])
" || tail -3 gpurun_out/ab_err.log
}
run "direct" X=1
[ -n "$AB_BASE" ] && run "direct (base library $AB_BASE)" LDPCB_LIBRARY=$AB_BASE
true
