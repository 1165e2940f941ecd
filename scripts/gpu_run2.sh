#!/bin/bash
# GPU session: parity tests, bench sweep over solver / n_chunk. Outputs land in gpurun_out/.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for cfg in "thomas 100" "pcr 16" "pcr 2" "pcr 4" "thomas 1" "pcr 64" "thomas 16"; do
  set -- $cfg
  timeout 300 python bench.py --solver $1 --n-chunk $2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --quiet-clocks >> gpurun_out/bench_sweep.jsonl 2>> gpurun_out/bench_sweep.err
done
timeout 600 python bench.py --solver pcr --n-chunk 4 --steps 3 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -3 gpurun_out/pytest_gpu.log; tail -c 3000 gpurun_out/bench_sweep.jsonl
