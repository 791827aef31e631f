#!/bin/bash
# compute-sanitizer pass over tools/sanitize_step.py (TMA and row-staging
# paths).  Summaries -> gpurun_out/sanitize_*.txt.  Usage: tools/gpu_sanitize.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for tma in 1 0; do
    env=""; [ $tma = 0 ] && env="CSZI_NO_TMA=1"
    out=gpurun_out/sanitize_${tool}_tma${tma}.txt
    env $env timeout 900 compute-sanitizer --tool $tool --print-limit 50 \
      python tools/sanitize_step.py > $out 2>&1
    echo "$tool tma=$tma rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ALL OK|FAILED' $out | tr '\n' ' ')"
  done
done
