#!/bin/bash
# Timing-only experiment builds of the library (wrong results by design):
# where the resident kernel's time goes. Run from the repo root:
#   bash scripts/exp_builds.sh build   # here (nvcc cross-compiles)
#   bash scripts/exp_builds.sh run     # on the GPU box
set -e
cd "$(dirname "$0")/.."
VARIANTS="NOFIX NOMUFU NOSYNC1"
if [ "$1" = build ]; then
  for v in $VARIANTS; do
    make -s -C paper_1202_1060_b200/csrc OBJ=obj_$v OUT=../libldpc_b200_$v.so EXTRA_NVFLAGS=-DLDPCB_EXP_$v >/dev/null
  done
  exit 0
fi
for rep in 1 2; do
  python scripts/exp_time.py base
  for v in $VARIANTS; do LDPCB_LIBRARY=paper_1202_1060_b200/libldpc_b200_$v.so python scripts/exp_time.py $v; done
done
