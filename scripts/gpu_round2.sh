#!/bin/bash
# Round-2 GPU evidence run: tests, the default two-leg bench line, reference arm,
# launch lists, ncu captures of both dominant kernels.
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=8 2>&1 | tail -40 > gpurun_out/gputest.log; tail -3 gpurun_out/gputest.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; cat gpurun_out/bench_c5.json
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/ref_c5.json 2> gpurun_out/ref_c5.err; cat gpurun_out/ref_c5.json
S1="python bench.py --workload c5_n1008 --frames 65536 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
S2="python bench.py --workload c5_n64800 --frames 8192 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$S1 > gpurun_out/s1.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5_n1008.csv $S1 > /dev/null 2>&1
$S2 > gpurun_out/s2.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5_n64800.csv $S2 > /dev/null 2>&1
$S1 > gpurun_out/s3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:decode_direct -s 1 -c 1 -f -o gpurun_out/prof_direct $S1 > gpurun_out/ncu1.log 2>&1
$S2 > gpurun_out/s4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stream_cn -s 45 -c 1 -f -o gpurun_out/prof_stream $S2 > gpurun_out/ncu2.log 2>&1
ls -la gpurun_out
cp profiles/dram_bytes_per_frame.json gpurun_out/dram_bytes_per_frame.json 2>/dev/null
python scripts/launch_summary.py gpurun_out/launches_c5_n1008.csv "C5 n=1008, 65536-frame decodes" 65536 c5_n1008 gpurun_out/dram_bytes_per_frame.json > gpurun_out/launches_c5_n1008.txt
python scripts/launch_summary.py gpurun_out/launches_c5_n64800.csv "C5 n=64800, one 8192-frame decode" 8192 c5_n64800 gpurun_out/dram_bytes_per_frame.json > gpurun_out/launches_c5_n64800.txt
cat gpurun_out/launches_c5_n1008.txt gpurun_out/launches_c5_n64800.txt
