#!/bin/bash
# Full ncu capture of one decode_direct launch (C5 n=1008 workload at 65536
# frames) and its text summaries (metrics, source-level stall hot spots).
mkdir -p gpurun_out
SMALL="python bench.py --workload c5_n1008 --frames 65536 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e ${SMALL_ARGS}"
$SMALL > gpurun_out/small.log 2>&1 || { cat gpurun_out/small.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:decode_direct -s 1 -c 1 -f -o gpurun_out/prof_dir $SMALL > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
ncu -i gpurun_out/prof_dir.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_dir_sass.csv 2>/dev/null
python scripts/ncu_hot.py gpurun_out/prof_dir_sass.csv 60 > gpurun_out/prof_dir_hot.txt 2>&1
bash scripts/ncu_summary.sh gpurun_out/prof_dir.ncu-rep gpurun_out/prof_dir > /dev/null 2>&1
cat gpurun_out/prof_dir.metrics.txt gpurun_out/prof_dir.sass_regions.txt
