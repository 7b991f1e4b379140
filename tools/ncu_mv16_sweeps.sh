#!/bin/bash
# ncu --set full of the 16-vector sweep kernels at C4 (one launch each after warm-up).
set -e
ncu --set full --import-source on --clock-control none --kernel-name-base function \
    -k regex:'k_(up_leaf|up_fused|down_fused|down_leaf)_mv' -s 12 -c 4 \
    -o gpurun_out/r02_mv16_sweeps python tools/mv16_time.py > /dev/null 2>&1
python profiles/summarize_ncu.py gpurun_out/r02_mv16_sweeps.ncu-rep > gpurun_out/r02_mv16_sweeps.txt
python tools/ncu_lines.py gpurun_out/r02_mv16_sweeps.ncu-rep 12 >> gpurun_out/r02_mv16_sweeps.txt
