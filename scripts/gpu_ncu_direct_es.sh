#!/bin/bash
# Full ncu capture of one early-stop decode_direct launch (C1 NDGSBP, 2.0 dB, <= 20 it) and its summaries.
mkdir -p gpurun_out
python scripts/es_decode.py 1048576 2.0 > gpurun_out/es.log 2>&1 || { cat gpurun_out/es.log; exit 1; }
python scripts/es_decode.py 1048576 1.5 >> gpurun_out/es.log 2>&1
cat gpurun_out/es.log
ncu --set full --clock-control none --import-source on -k regex:decode_direct -s 1 -c 1 -f -o gpurun_out/prof_es python scripts/es_decode.py 131072 2.0 > gpurun_out/ncu_es.log 2>&1
tail -2 gpurun_out/ncu_es.log
ncu -i gpurun_out/prof_es.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_es_sass.csv 2>/dev/null
python scripts/ncu_hot.py gpurun_out/prof_es_sass.csv 60 > gpurun_out/prof_es_hot.txt 2>&1
bash scripts/ncu_summary.sh gpurun_out/prof_es.ncu-rep gpurun_out/prof_es > /dev/null 2>&1
cat gpurun_out/prof_es.metrics.txt gpurun_out/prof_es.sass_regions.txt
