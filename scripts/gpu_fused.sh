# fused-loss / static-VJP check: new tests, the headline parity tests, a short bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_loss.py tests/test_gpu_headline.py -x -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/fused_bench.json 2> gpurun_out/fused_bench.err
python - <<'P'
import json; d=json.loads(open("gpurun_out/fused_bench.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["value"], d["kernel_ms_per_step"], d["gpu_launches"], d["parity"]["ok"], d["e2e"]["value"])
print(d["c2_solver_family"])
P
