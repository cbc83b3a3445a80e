#!/bin/bash
# Summarise an ncu report into profiles/: key metrics + per-region SASS mix.
# usage: scripts/ncu_summary.sh gpurun_out/prof.ncu-rep profiles/r01_name
rep=$1; out=$2
ncu -i "$rep" --page details --csv > "$out.details.csv" 2>/dev/null
ncu -i "$rep" --page raw --csv 2>/dev/null | python3 -c "
import csv, sys
rows = list(csv.reader(sys.stdin))
hdr, units, vals = rows[0], rows[1], rows[2:]
keys = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__inst_executed.sum',
        'smsp__inst_executed.avg.per_cycle_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'launch__registers_per_thread', 'launch__block_size', 'launch__grid_size', 'sm__cycles_elapsed.avg.per_second']
for v in vals:
    for k in keys:
        if k in hdr:
            i = hdr.index(k); print(f'{k:70s} {units[i]:>12s} {v[i]}')
" > "$out.metrics.txt"
ncu -i "$rep" --page source --csv --print-source sass > /tmp/_sass.csv 2>/dev/null && python3 scripts/ncu_sass_summary.py /tmp/_sass.csv > "$out.sass_regions.txt"
cat "$out.metrics.txt" "$out.sass_regions.txt"
