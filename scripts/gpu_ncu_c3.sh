#!/bin/bash
# Full ncu capture of one C3 decode (posterior-based resident kernel, 16-wide bucket) and its summaries.
mkdir -p gpurun_out
python scripts/c3_decode.py 65536 > gpurun_out/c3.log 2>&1 || { cat gpurun_out/c3.log; exit 1; }
cat gpurun_out/c3.log
ncu --set full --clock-control none --import-source on -k regex:decode_ -s 1 -c 1 -f -o gpurun_out/prof_c3 python scripts/c3_decode.py 65536 > gpurun_out/ncu_c3.log 2>&1
tail -2 gpurun_out/ncu_c3.log
ncu -i gpurun_out/prof_c3.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_c3_sass.csv 2>/dev/null
python scripts/ncu_hot.py gpurun_out/prof_c3_sass.csv 40 > gpurun_out/prof_c3_hot.txt 2>&1
bash scripts/ncu_summary.sh gpurun_out/prof_c3.ncu-rep gpurun_out/prof_c3 > /dev/null 2>&1
cat gpurun_out/prof_c3.metrics.txt gpurun_out/prof_c3.sass_regions.txt
head -1 gpurun_out/prof_c3_sass.csv | tr ',' '\n' | head -80
