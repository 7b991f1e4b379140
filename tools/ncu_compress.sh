#!/bin/bash
# ncu --set full of the compression kernels at C3 (3D n=2^20, k=64, eps=1e-6),
# one launch each (the largest level), summarised to text under gpurun_out/.
set -e
cfg="3 1048576 4 1e-6"
run() {  # name regex skip
  ncu --set full --import-source on --clock-control none --kernel-name-base function -k "regex:$2" -s "$3" -c 1 \
      -o "gpurun_out/$1" python tools/compress_profile.py $cfg > /dev/null 2>&1
  python profiles/summarize_ncu.py "gpurun_out/$1.ncu-rep" > "gpurun_out/$1.txt"
  python tools/ncu_lines.py "gpurun_out/$1.ncu-rep" 20 >> "gpurun_out/$1.txt"
}
run r01_k_weights_leaf '^k_weights$' 13      # level 14 (16384 nodes)
run r01_k_project_orth '^k_project$' 0
run r01_k_project_trunc '^k_project$' 1
run r01_k_jacobi64_leaf '^k_jacobi64$' 0
run r01_k_orth_level14 '^k_orth_level$' 0
run r01_k_trunc_level_pre14 '^k_trunc_level_pre$' 0
rm -f gpurun_out/r01_k_project_*.ncu-rep gpurun_out/r01_k_jacobi64_leaf.ncu-rep gpurun_out/r01_k_orth_level14.ncu-rep gpurun_out/r01_k_trunc_level_pre14.ncu-rep
ls -la gpurun_out
