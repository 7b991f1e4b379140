#!/bin/bash
# ncu --set full of the fused dataflow sweeps of the n=2^22 mat-vec (bench workload).
for k in k_up_fused k_down_fused; do
  ncu --set full --import-source on --clock-control none --kernel-name-base function -k "regex:^$k$" -s 2 -c 1 \
      -o gpurun_out/r01_$k python bench.py --steps 3 --warmup 3 --no-compress --no-cpu-baseline > /dev/null 2>&1
  python profiles/summarize_ncu.py gpurun_out/r01_$k.ncu-rep > gpurun_out/r01_$k.txt
  rm -f gpurun_out/r01_$k.ncu-rep
done
