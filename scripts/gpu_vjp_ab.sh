set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_v2.py -x -q -m gpu 2>&1 | tail -5
for v in "" variants/vjp_gen.so variants/vjp_minb2.so "" variants/vjp_gen.so variants/vjp_minb2.so; do
  CKO_LIB_PATH=$v timeout 300 python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', d['ms_per_step'], d['value'])"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:vjp -c 6 python bench.py --steps 2 --warmup 3 2>&1 | grep -E "vjp|gpu__time" | head -12
CKO_LIB_PATH=variants/vjp_gen.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:vjp -c 6 python bench.py --steps 2 --warmup 3 2>&1 | grep -E "vjp|gpu__time" | head -12
