#!/bin/bash
# ncu --set full of k_project (orth: launch 0, trunc: launch 1) at C3.
cfg="3 1048576 4 1e-6"
for s in 0 1; do
  ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:^k_project$ -s $s -c 1 \
      -o gpurun_out/kp$s python tools/compress_profile.py $cfg > /dev/null 2>&1
  python profiles/summarize_ncu.py gpurun_out/kp$s.ncu-rep > gpurun_out/kp$s.txt
  python tools/ncu_lines.py gpurun_out/kp$s.ncu-rep 25 >> gpurun_out/kp$s.txt
  ncu -i gpurun_out/kp$s.ncu-rep --page raw --csv > gpurun_out/kp${s}_raw.csv
  rm -f gpurun_out/kp$s.ncu-rep
done
