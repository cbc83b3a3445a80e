#!/bin/bash
# One GPU call: bench, launch list, one full ncu capture of the decode kernel.
set -x
SMALL="python bench.py --frames 65536 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e ${SMALL_ARGS}"
python bench.py --steps 5 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -2 gpurun_out/bench.err
cat gpurun_out/bench.json
$SMALL > gpurun_out/small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launches.log 2>&1
$SMALL > gpurun_out/small2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:decode_resident -s 1 -c 1 -f -o gpurun_out/prof $SMALL > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
