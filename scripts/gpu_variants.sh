#!/bin/bash
# Bench A/B variants built by scripts/build_variant.sh: VARIANTS="a b" NCS="100" bash scripts/gpu_variants.sh
for v in ${VARIANTS:-base}; do
  for nc in ${NCS:-100}; do
    lib=""; [ "$v" != base ] && lib="variants/$v.so"
    CKO_LIB_PATH=$lib timeout 300 python bench.py --solver thomas --n-chunk $nc --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-c3 --quiet-clocks 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['n_chunk'], '%.4g'%d['value'], {k: round(v, 2) for k, v in d['kernel_ms_per_step'].items()})"
  done
done
