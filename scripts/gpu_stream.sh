# streamed time grid: tests, then bench e2e with and without streaming
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_loss.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -8
for v in 0 1 0 1; do
  CKO_NO_TIME_STREAM=$v timeout 600 python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 > gpurun_out/stream_$v.json
  python -c "import json; d=json.load(open('gpurun_out/stream_$v.json')); print('no_stream=$v', d['ms_per_step'], d['value'], 'e2e', d['e2e']['ms_per_step'], d['e2e']['value'])"
done
