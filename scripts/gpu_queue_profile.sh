#!/bin/bash
# ncu launch list of one C4 early-stop decode through the streamed frame queue. Keep it small: ncu
# serialises every launch (16384 frames on 8192 lanes = 125 iterations, 12 000 launches, about 5 minutes;
# 32768 frames on 4096 lanes did not finish in 25).
mkdir -p gpurun_out
F=${1:-16384}
export LDPCB_STREAM_CHUNK=${2:-8192}
python scripts/c4_queue_profile.py $F > gpurun_out/q.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4_queue.csv python scripts/c4_queue_profile.py $F > /dev/null 2>&1
cat gpurun_out/q.log
python scripts/launch_summary.py gpurun_out/launches_c4_queue.csv "C4 early stop <= 30 it from the frame queue, $F frames on $LDPCB_STREAM_CHUNK lanes" 2>&1 | head -20
