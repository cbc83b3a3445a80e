#!/bin/bash
# A/B of two builds of the library on the C1 workloads (scripts/ab_speed.py):
# the in-tree build against paper_1202_1060_b200/libldpc_b200_base.so.
for rep in 1 2; do
  LDPCB_LIBRARY=paper_1202_1060_b200/libldpc_b200_base.so python scripts/ab_speed.py 2>&1 | grep "${AB_FILTER:-it=10}"
  python scripts/ab_speed.py 2>&1 | grep "${AB_FILTER:-it=10}"
done
