#!/bin/bash
# Round-end evidence: GPU test suite, smoke(), default bench, launch lists
# (512^3 and RTM) and ncu --set full summaries of the top kernels.
# Usage: tools/gpu_final.sh TAG
tag=${1:-r02f}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -rfE > gpurun_out/${tag}_pytest_gpu.txt 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/${tag}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1
echo "smoke rc=$?"; tail -1 gpurun_out/${tag}_smoke.txt
bash tools/gpu_round.sh ${tag}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_rtm.csv python tools/profile_step.py 449,449,235 > /dev/null 2>&1
python tools/launches.py gpurun_out/${tag}_launches_rtm.csv > gpurun_out/${tag}_launches_rtm.txt
