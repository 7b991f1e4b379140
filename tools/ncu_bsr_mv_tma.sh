#!/bin/bash
# ncu --set full of the TMA-fed 16-vector coupling kernel at C4 (one launch).
set -e
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_bsr_mv -c 1 \
    -o gpurun_out/bsr_tma python tools/mv16_timeline.py 1 > /dev/null 2>&1



