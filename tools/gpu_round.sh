#!/bin/bash
# Round evidence: full bench (JSON), launch list of one compress+decompress
# step, ncu --set full summaries of the top kernels.  Usage: tools/gpu_round.sh tag
tag=${1:-r01}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/${tag}_bench.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv python tools/profile_step.py > /dev/null 2>&1
python tools/launches.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launches.txt
NCU_SKIP=2 bash tools/gpu_ncu.sh ${tag} k_t3_predict k_t3_reconstruct k_enc_nz_emit k_enc_nz_count k_dec_write_zr k_dec_spec k_range k_p2d_tables k_p2d_expand k_codebook
