#!/bin/bash
# A/B of libcszi builds (tools/t3_time.py per build) + selected GPU tests on
# the last one.  Usage: tools/gpu_ab.sh "pytest -k expr" a.so b.so ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
sel=$1; shift
for lib in "$@"; do
  echo "== $lib"
  CSZI_LIB=$lib timeout 600 python tools/t3_time.py $AB_SHAPES 2>&1 | tail -8
done
if [ -n "$sel" ]; then
  timeout 1200 python -m pytest tests -q -m gpu -x $sel > gpurun_out/ab_pytest.txt 2>&1
  echo "pytest rc=$?"; tail -3 gpurun_out/ab_pytest.txt
fi
