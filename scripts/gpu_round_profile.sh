#!/bin/bash
# Round profile: full bench line, ncu launch list of one bench step, full ncu
# captures of the forward / adjoint kernels at the bench configuration.
TAG=${1:-r1v2}
ARGS=${2:-"--solver thomas --n-chunk 100"}
mkdir -p gpurun_out
timeout 900 python bench.py $ARGS > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py $ARGS --steps 1 --warmup 1 \
  --no-e2e --no-cpu-baseline --no-c3 --quiet-clocks > /dev/null 2>&1
for K in fwd adj; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${K}(2|_pcr2)?_kernel" -c 1 \
    -o gpurun_out/${TAG}_${K} -f python bench.py $ARGS --steps 1 --warmup 0 \
    --no-e2e --no-cpu-baseline --no-c3 --quiet-clocks > gpurun_out/${TAG}_${K}.log 2>&1
done
cat gpurun_out/${TAG}_bench.json | head -c 3000; tail -3 gpurun_out/${TAG}_bench.err
ls gpurun_out
