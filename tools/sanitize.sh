#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py -> gpurun_out/r02_sanitizer.txt
out=gpurun_out/r02_sanitizer.txt
echo "# compute-sanitizer on tools/sanitize_run.py (construct, hmv, 16-vector, phases, compress 2D/3D, non-symmetric, blocks > 64, one-call partitioned hmv / 16-vector, async host calls), B200" > $out
for tool in memcheck racecheck synccheck; do
  echo "## $tool" >> $out
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py 2>&1 | grep -E "COMPUTE-SANITIZER|ERROR SUMMARY|RACECHECK SUMMARY|^ok|Error|Hazard|hazard" | head -40 >> $out
  echo "rc=${PIPESTATUS[0]}" >> $out
done
