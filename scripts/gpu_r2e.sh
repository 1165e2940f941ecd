#!/bin/bash
# Round-2 final measurement of the structured kernels: bench line, launch list, ncu captures, line stalls, traffic.
mkdir -p gpurun_out
T=${TAG:-r2e}
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
TAG=$T bash scripts/gpu_sp_profile.sh > gpurun_out/${T}_profile.log 2>&1
tail -c 600 gpurun_out/${T}_bench.json; tail -2 gpurun_out/${T}_bench.err
