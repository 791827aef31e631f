#!/bin/bash
# one GPU round trip: tests, bench, launch list (+ optional ncu of a kernel)
cd "$(dirname "$0")/.."
OUT=gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.txt 2>&1
tail -2 $OUT/pytest_gpu.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench.json 2> $OUT/bench.err
tail -2 $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/profile_step.py > /dev/null 2>&1
if [ -n "$NCU_KERNEL" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$NCU_KERNEL -s ${NCU_SKIP:-2} -c 1 -o $OUT/prof_$NCU_KERNEL python tools/profile_step.py > $OUT/ncu_full.txt 2>&1
fi
