#!/bin/bash
# Full GPU pass on the tree: smoke, the -m gpu suite, the one-GPU two-rank bench plumbing, one bench line.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
CKO_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench2 rc=$?" >> gpurun_out/bench2.err
tail -3 gpurun_out/smoke.log; tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench2.err; tail -c 800 gpurun_out/bench2.json
