#!/bin/bash
# ncu --set full of the 16-vector coupling kernel k_bsr_mv at C4 (n = 2^22, 16 vectors),
# one launch after warm-up, summarised to gpurun_out/r01_k_bsr_mv.txt.
set -e
ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:'^k_bsr_mv$' -s 3 -c 1 \
    -o gpurun_out/r01_k_bsr_mv python tools/mv16_time.py > /dev/null 2>&1
python profiles/summarize_ncu.py gpurun_out/r01_k_bsr_mv.ncu-rep > gpurun_out/r01_k_bsr_mv.txt
python tools/ncu_lines.py gpurun_out/r01_k_bsr_mv.ncu-rep 15 >> gpurun_out/r01_k_bsr_mv.txt
ncu -i gpurun_out/r01_k_bsr_mv.ncu-rep --page raw --csv --metrics sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum > gpurun_out/r01_k_bsr_mv_pipe.csv
rm -f gpurun_out/r01_k_bsr_mv.ncu-rep
