#!/bin/bash
# One full ncu capture of a named kernel from a short bench run: TAG KERNEL_REGEX BENCH_ARGS
TAG=$1; K=$2; shift 2
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 \
  -o gpurun_out/${TAG} -f python bench.py "$@" --steps 1 --warmup 0 \
  --no-e2e --no-cpu-baseline --quiet-clocks > gpurun_out/${TAG}.log 2>&1
tail -3 gpurun_out/${TAG}.log
