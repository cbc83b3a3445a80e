#!/bin/bash
# A/B of early-stop decoding from a frame queue (LDPCB_FRAME_QUEUE=0: one
# frame set per CTA) on C1 (2^20 frames, 2.0 dB, <= 20 it) and C3.
for q in 0 1; do
  echo "LDPCB_FRAME_QUEUE=$q"
  LDPCB_FRAME_QUEUE=$q python scripts/ab_speed.py 2>&1 | grep "es=True"
  LDPCB_FRAME_QUEUE=$q python scripts/c3_speed.py 2>&1 | grep "es=True"
done
