#!/bin/bash
# Run the reference (oracle/_ref) at every config on a gpurun box:
#   gpurun --timeout 3000 -- bash tools/run_config_golden.sh [CASES...]
# Output: gpurun_out/config_golden/<case>.{json,npz,log}
OUT=gpurun_out/config_golden
mkdir -p $OUT
CASES=${@:-C1 C1k64 C2 C2alt C4 C3}
for c in $CASES; do
  timeout 2400 python tests/golden/make_config_golden.py --case $c --out $OUT > $OUT/$c.log 2>&1
  echo "$c rc=$?" | tee -a $OUT/status.txt
  tail -3 $OUT/$c.log
done
free -g > $OUT/free.txt
