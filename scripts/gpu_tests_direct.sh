#!/bin/bash
python -m pytest tests -m gpu -q -x --durations=5 -k "not c4_long and not stream" 2>&1 | tail -8
bash scripts/direct_ab.sh 2>&1 | grep direct
AB_KERNEL=0 python scripts/ab_speed.py 2>&1 | grep frames/s | cut -c1-100
