# A/B of kernel variants at the bench dt (1e-6: one row exchange per forward block) and at dt = 5e-5 (exchanges in most columns); VARS="base x" bash scripts/gpu_cmp_dt.sh
for v in ${VARS:-base x2}; do
  lib=""; [ "$v" != base ] && lib="variants/$v.so"
  for a in "--nb 1000 --nt 10000 --n-chunk 100" "--nb 1000 --nt 200 --n-chunk 100"; do
    CKO_LIB_PATH=$lib timeout 300 python bench.py $a --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-c3 --quiet-clocks 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); c=d['config']; print('$v', c['n_time'], '%.4g'%d['value'], {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()})"
  done
done
[ -n "$TESTLIB" ] && CKO_LIB_PATH=$TESTLIB timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
