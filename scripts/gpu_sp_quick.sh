#!/bin/bash
# structured kernels: their tests, the MDS v2 tests, one bench line
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_structured.py -x -q --timeout 120 > gpurun_out/sp1.log 2>&1; echo "rc=$?" >> gpurun_out/sp1.log
timeout 900 python -m pytest tests/test_gpu_v2.py tests/test_gpu_headline.py -x -q --timeout 300 -k "mds" > gpurun_out/sp2.log 2>&1; echo "rc=$?" >> gpurun_out/sp2.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-c3 > gpurun_out/sp_bench.json 2> gpurun_out/sp_bench.err; echo "rc=$?" >> gpurun_out/sp_bench.err
tail -4 gpurun_out/sp1.log; tail -3 gpurun_out/sp2.log; tail -3 gpurun_out/sp_bench.err
python - <<'PY'
import json
for l in open('gpurun_out/sp_bench.json'):
    if l.startswith('{"metric'):
        d=json.loads(l); print(d['value'], d['ms_per_step'], d['kernel_ms_per_step'], d['parity']['ok'], d['e2e']['value'])
PY
