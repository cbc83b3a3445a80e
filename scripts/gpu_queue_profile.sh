#!/bin/bash
mkdir -p gpurun_out
export LDPCB_STREAM_CHUNK=8192; python scripts/c4_queue_profile.py 16384 > gpurun_out/q.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4_queue.csv python scripts/c4_queue_profile.py 16384 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_c4_queue.csv "C4 queue" 2>&1 | head -20
