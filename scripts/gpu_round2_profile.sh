#!/bin/bash
# Round-2 profile: the default bench line, ncu launch list of one bench step, full ncu captures of the
# forward / adjoint Thomas kernels at the bench configuration, the C4 DMMA evaluation kernel (tensor pipe),
# the n = 20 PCR kernels (C2, short grid). Everything into gpurun_out/r2_*.
mkdir -p gpurun_out
T=r2
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 1 \
  --no-e2e --no-cpu-baseline --no-c3 --quiet-clocks > /dev/null 2>&1
for K in fwd adj; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${K}2_kernel" -c 1 \
    -o gpurun_out/${T}_${K} -f python bench.py --steps 1 --warmup 0 \
    --no-e2e --no-cpu-baseline --no-c3 --quiet-clocks > gpurun_out/${T}_${K}.log 2>&1
done
timeout 900 ncu --set full --clock-control none -k regex:"node_eval_kernel" -s 20 -c 1 \
  -o gpurun_out/${T}_node_eval -f python scripts/c4_bench.py 0,20 > gpurun_out/${T}_node_eval.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_c4_launches.csv python scripts/c4_bench.py 0,20 > /dev/null 2>&1
NT=400 timeout 900 ncu --set full --clock-control none -k regex:"(fwd|adj)_pcrw_kernel" -c 2 \
  -o gpurun_out/${T}_pcrw -f python scripts/c2_pcr_sweep.py pcr,100,1000 > gpurun_out/${T}_pcrw.log 2>&1
tail -c 2500 gpurun_out/${T}_bench.json; tail -3 gpurun_out/${T}_bench.err
ls -la gpurun_out | head -40
