#!/bin/bash
# GPU test pass: the full -m gpu suite (log in gpurun_out/pytest_gpu.txt),
# then a short bench line.  Usage: tools/gpu_tests.sh [pytest args...]
cd "$(dirname "$0")/.."
OUT=gpurun_out
mkdir -p $OUT
timeout 2400 python -m pytest tests -q -m gpu -rfE "$@" > $OUT/pytest_gpu.txt 2>&1
echo "pytest rc=$?"
tail -25 $OUT/pytest_gpu.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"
tail -c 1500 $OUT/bench.json
tail -5 $OUT/bench.err
