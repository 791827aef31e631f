#!/bin/bash
# A/B of two builds of libcszi.so on one box: per-kernel ncu times of one
# warm compress+decompress step and bench ms.  Usage: tools/ab.sh a.so b.so
for lib in "$@"; do
  echo "== $lib"
  CSZI_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ab.csv python tools/profile_step.py > /dev/null 2>&1
  python tools/launches.py gpurun_out/ab.csv 2>/dev/null | head -${AB_LINES:-20}
  CSZI_LIB=$lib timeout 300 python bench.py --steps 30 --warmup 3 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('bench', d['ms_per_step'], d['decompress_ms_per_step'])"
done
