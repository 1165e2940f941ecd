#!/bin/bash
# Quick loop for kernel work: v2 parity tests, C2 bench at n_chunk 100 / 32, forward trace of CTA 0.
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests/test_gpu_v2.py -x -q 2>&1 | tail -3
fi
for nc in ${NCS:-100 32}; do
  timeout 300 python bench.py --solver thomas --n-chunk $nc --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-c3 --quiet-clocks 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['n_chunk'], '%.4g'%d['value'], {k: round(v, 2) for k, v in d['kernel_ms_per_step'].items()})"
done
[ -n "$TRACE" ] && timeout 120 python scripts/trace_v2.py 1000 400 100 > gpurun_out/trace.txt 2>&1; [ -n "$TRACE" ] && grep -v "^[0-9]* \s*[0-9.]* \s*[0-9.]* " gpurun_out/trace.txt | tail -20
true
