#!/bin/bash
# Quick GPU check of the generation-2 kernels: parity tests + short benches.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_v2.py -x -q > gpurun_out/v2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/v2_pytest.log
tail -15 gpurun_out/v2_pytest.log
for cfg in ${V2CFGS:-"thomas 100" "thomas 16" "thomas 1"}; do
  set -- $cfg
  timeout 300 python bench.py --solver $1 --n-chunk $2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --quiet-clocks >> gpurun_out/v2_bench.jsonl 2>> gpurun_out/v2_bench.err
done
python - <<'P'
import json
for l in open("gpurun_out/v2_bench.jsonl"):
    d=json.loads(l); print(d["config"]["solver"], d["config"]["n_chunk"], "%.3g"%d["value"], d["ms_per_step"], d["kernel_ms_per_step"])
P
tail -5 gpurun_out/v2_bench.err
