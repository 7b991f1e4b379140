#!/bin/bash
cfg="3 1048576 4 1e-6"
run() {
  ncu --set full --import-source on --clock-control none --kernel-name-base function -k "regex:$2" -s "$3" -c 1 \
      -o "gpurun_out/$1" python tools/compress_profile.py $cfg > /dev/null 2>&1
  python profiles/summarize_ncu.py "gpurun_out/$1.ncu-rep" > "gpurun_out/$1.txt"
  python tools/ncu_lines.py "gpurun_out/$1.ncu-rep" 30 >> "gpurun_out/$1.txt"
  ncu -i "gpurun_out/$1.ncu-rep" --page details --csv > "gpurun_out/$1.details.csv" 2>/dev/null
  rm -f "gpurun_out/$1.ncu-rep"
}
run r01_k_orth_level14b '^k_orth_level$' 0
run r01_k_trunc_level_pre14b '^k_trunc_level_pre$' 0
