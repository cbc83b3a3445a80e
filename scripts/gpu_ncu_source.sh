#!/bin/bash
# Full ncu capture of one decode_resident launch + its SASS source page.
SMALL="python bench.py --frames 65536 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e ${SMALL_ARGS}"
$SMALL > gpurun_out/small.log 2>&1 || { cat gpurun_out/small.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:decode_resident -s 1 -c 1 -f -o gpurun_out/prof $SMALL > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
ncu -i gpurun_out/prof.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_sass.csv 2>/dev/null
ls -la gpurun_out/
