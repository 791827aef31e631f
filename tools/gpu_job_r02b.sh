set -x
bash tools/gpu_sanitize.sh
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_512cube.csv python tools/profile_step.py > /dev/null 2>&1
python tools/launches.py gpurun_out/r02b_launches_512cube.csv > gpurun_out/r02b_launches_512cube.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_rtm.csv python tools/profile_step.py 449,449,235 > /dev/null 2>&1
python tools/launches.py gpurun_out/r02b_launches_rtm.csv > gpurun_out/r02b_launches_rtm.txt
NCU_SKIP=2 bash tools/gpu_ncu.sh r02b k_t3_predict k_t3_reconstruct
SHAPE=449,449,235 NCU_SKIP=2 bash tools/gpu_ncu.sh r02b_rtm k_t3_predict k_t3_reconstruct
