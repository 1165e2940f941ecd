#!/bin/bash
# Round-2 close: smoke, the -m gpu suite, the default bench line, launch list of one bench step.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc=$?" >> gpurun_out/r2f_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2f_launches.csv python bench.py --steps 1 --warmup 1 \
  --no-e2e --no-cpu-baseline --no-c3 --quiet-clocks > /dev/null 2>&1
tail -2 gpurun_out/smoke.log; tail -2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/r2f_bench.err
