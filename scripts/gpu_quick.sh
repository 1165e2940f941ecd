# quick guarded check: one small case with a hard per-test timeout, then the A/B if it passed
timeout 300 python -m pytest tests/test_gpu_fused_loss.py -x -q -m gpu --timeout 60 -k "mds20-thomas" 2>&1 | tail -4 || exit 1
timeout 900 python -m pytest ${AB_TESTS:-tests/test_gpu_fused_loss.py} -x -q -m gpu --timeout 120 2>&1 | tail -4
