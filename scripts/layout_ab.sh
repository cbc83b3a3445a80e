#!/bin/bash
# A/B of the bank-layout annealing effort (LDPCB_BANK_ITERS moves per CN; 0 = no colouring)
mkdir -p gpurun_out
for it in ${ITERS:-0 1000 4000 20000}; do
  echo "== LDPCB_BANK_ITERS=$it"
  LDPCB_BANK_ITERS=$it python scripts/ab_speed.py 2>&1 | grep -v "^$"
done
