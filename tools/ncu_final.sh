#!/bin/bash
# ncu --set full of the compression kernels at C3 (3D n=2^20, k=64, eps=1e-6)
# in their final form, one launch each (the largest level), summarised to
# text under gpurun_out/ (reports deleted: the 64 MiB return limit).
cfg="3 1048576 4 1e-6"
run() {  # name regex skip
  ncu --set full --import-source on --clock-control none --kernel-name-base function -k "regex:$2" -s "$3" -c 1 \
      -o "gpurun_out/$1" python tools/compress_profile.py $cfg > /dev/null 2>&1
  python profiles/summarize_ncu.py "gpurun_out/$1.ncu-rep" > "gpurun_out/$1.txt"
  python tools/ncu_lines.py "gpurun_out/$1.ncu-rep" 20 >> "gpurun_out/$1.txt"
  rm -f "gpurun_out/$1.ncu-rep"
}
# launch indices from a gpu__time_duration pass: k_project 0..10 = orth levels
# 14..4, 11..21 = truncation levels 14..4; k_weights 18 = level 14
[ -n "$ONLY" ] || {
run r01f_k_orth_level14 '^k_orth_level$' 0
run r01f_k_project_orth14 '^k_project$' 0
run r01f_k_trunc_leaf_pre '^k_trunc_leaf_pre$' 0
run r01f_k_jacobi64_leaf '^k_jacobi64$' 0
run r01f_k_trunc_level_pre14 '^k_trunc_level_pre$' 0
}
run r01f_k_weights_leaf '^k_weights$' 18
run r01f_k_project_trunc14 '^k_project$' 11
ls -la gpurun_out | grep r01f
