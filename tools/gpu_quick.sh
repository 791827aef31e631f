#!/bin/bash
# GPU-box iteration helper: gpu tests, a short bench, and the ncu launch list
# of one compress+decompress step (tools/profile_step.py).  Usage: tag [pytest-args]
tag=${1:-q}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_reference_suite.py::test_reference_suite_passes_against_facade "$@" > gpurun_out/${tag}_pytest.txt 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/${tag}_pytest.txt
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/${tag}_bench.json'));print('compress',d['value'],'ms',d['ms_per_step'],'decomp',d['decompress_gbs'],'ms',d['decompress_ms_per_step'],'parity',d.get('parity_vs_oracle'),'e2e',d['e2e']['value'],d['e2e_decompress']['value'])" || tail -20 gpurun_out/${tag}_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv python tools/profile_step.py > /dev/null 2>&1
python tools/launches.py gpurun_out/${tag}_launches.csv | tee gpurun_out/${tag}_launches.txt
