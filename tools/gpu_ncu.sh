#!/bin/bash
# ncu --set full capture of named kernels in one compress+decompress step.
# Usage: tools/gpu_ncu.sh tag kernel_regex [kernel_regex ...]
tag=$1; shift
mkdir -p gpurun_out
for k in "$@"; do
  name=$(echo "$k" | tr -cd 'a-zA-Z0-9_')
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:$k" -s 2 -c 1 \
    -o gpurun_out/${tag}_${name} -f python tools/profile_step.py > gpurun_out/${tag}_${name}.log 2>&1
  echo "ncu $k rc=$?"
done
