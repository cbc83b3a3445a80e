#!/bin/bash
# A/B of the posterior-free resident kernel (direct.cu) against decode_resident
# on the C5 n=1008 bench workload: smoke parity first, then kernel-only rates.
mkdir -p gpurun_out
python __graft_entry__.py smoke 2>&1 | tail -2
B="python bench.py --workload c5_n1008 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
run() { # label, env..., args
  local label=$1; shift
  env "$@" $B $EXTRA 2> gpurun_out/ab_err.log | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l)
        print('$label', 'ms', round(d['ms_per_step'], 3), 'frac', round(d['roofline']['frac'], 4), 'plan', d['config']['plan'], 'FER', d['counters']['frame_errors'] / d['counters']['frames'], 'BE', d['counters']['bit_errors'])
" || tail -3 gpurun_out/ab_err.log
}
EXTRA="--kernel 1"; run resident X=1; EXTRA=""
run "direct staged records" LDPCB_BANK_ITERS=4000
run "direct register records" LDPCB_BANK_ITERS=4000 LDPCB_LIBRARY=paper_1202_1060_b200/libldpc_b200_regrec.so
