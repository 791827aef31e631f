#!/bin/bash
# ncu --set full capture of named kernels in one compress+decompress step
# (tools/profile_step.py); summaries are written on the box, reports kept
# only when KEEP_REP=1 (they are large).  Usage: tools/gpu_ncu.sh tag regex...
tag=$1; shift
mkdir -p gpurun_out
for k in "$@"; do
  name=$(echo "$k" | tr -cd 'a-zA-Z0-9_')
  rep=gpurun_out/${tag}_${name}
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:$k" -s ${NCU_SKIP:-2} -c 1 \
    -o $rep -f python tools/profile_step.py ${SHAPE:-} > ${rep}.log 2>&1
  echo "ncu $k rc=$?"
  python tools/ncu_summary.py ${rep}.ncu-rep 40 > ${rep}.txt 2>&1
  ncu -i ${rep}.ncu-rep --page source --csv --print-source sass > ${rep}.sass.csv 2>/dev/null
  [ "${KEEP_REP:-0}" = 1 ] || rm -f ${rep}.ncu-rep
done
