#!/bin/bash
# Per-launch duration, FP64 / DMMA pipe utilisation and DRAM throughput of every kernel of
# one compress() at C3 (3D n=2^20, k=64, eps=1e-6) -> gpurun_out/r01_compress_pipes.csv;
# tools/compress_pipes_summary.py turns it into profiles/tensor_pipe.json's compression_C3.
ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv --log-file gpurun_out/r01_compress_pipes.csv \
    python tools/compress_profile.py 3 1048576 4 1e-6 > /dev/null 2>&1
