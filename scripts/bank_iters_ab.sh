#!/bin/bash
# Annealing effort of the bank colouring (LDPCB_BANK_ITERS moves per CN) on the C5 n=1008 bench workload.
mkdir -p gpurun_out
B="python bench.py --workload c5_n1008 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
for it in "$@"; do
  t0=$(date +%s)
  LDPCB_BANK_ITERS=$it $B 2> gpurun_out/e.log | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('moves per CN $it: ms', round(d['ms_per_step'], 3), 'frac', round(d['roofline']['frac'], 4))
"
  echo "  wall $(( $(date +%s) - t0 )) s"
done
