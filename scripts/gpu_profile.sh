#!/bin/bash
# GPU session: ncu launch list of one bench step + one full ncu capture of the
# forward and adjoint kernels. Outputs land in gpurun_out/ (TAG = round tag).
TAG=${1:-r1}
ARGS=${2:-"--solver thomas --n-chunk 16"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py $ARGS --steps 1 --warmup 1 \
  --no-e2e --no-cpu-baseline --quiet-clocks > gpurun_out/${TAG}_launches_bench.log 2>&1
for K in fwd_kernel adj_kernel; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 \
  -o gpurun_out/${TAG}_$K -f python bench.py $ARGS --nt 2000 --steps 1 --warmup 0 \
  --no-e2e --no-cpu-baseline --quiet-clocks > gpurun_out/${TAG}_$K.log 2>&1
done
ls -la gpurun_out
