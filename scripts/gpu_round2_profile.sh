#!/bin/bash
# Round-2 profile: the default bench line, ncu launch list of one bench step, full ncu captures of the
# forward / adjoint Thomas kernels at the bench configuration, the C4 DMMA evaluation kernel (tensor pipe),
# the n = 20 PCR kernels (C2, short grid). Summaries are written on the box (the .ncu-rep files are too
# large to travel back and are deleted): gpurun_out/r2_*.
mkdir -p gpurun_out
T=${TAG:-r2}
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 1 \
  --no-e2e --no-cpu-baseline --no-c3 --quiet-clocks > /dev/null 2>&1
mkdir -p /tmp/reps
for K in fwd adj; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${K}2_kernel" -c 1 \
    -o /tmp/reps/${T}_${K} -f python bench.py --steps 1 --warmup 0 \
    --no-e2e --no-cpu-baseline --no-c3 --quiet-clocks > gpurun_out/${T}_${K}.log 2>&1
done
timeout 900 ncu --set full --clock-control none -k regex:"node_eval_kernel" -s 20 -c 1 \
  -o /tmp/reps/${T}_node_eval -f python scripts/c4_bench.py 0,20 > gpurun_out/${T}_node_eval.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_c4_launches.csv python scripts/c4_bench.py 0,20 > /dev/null 2>&1
NT=400 timeout 900 ncu --set full --clock-control none -k regex:"(fwd|adj)_pcrw_kernel" -c 2 \
  -o /tmp/reps/${T}_pcrw -f python scripts/c2_pcr_sweep.py pcr,100,1000 > gpurun_out/${T}_pcrw.log 2>&1
python scripts/ncu_summary.py /tmp/reps/${T}_fwd.ncu-rep /tmp/reps/${T}_adj.ncu-rep /tmp/reps/${T}_node_eval.ncu-rep \
  /tmp/reps/${T}_pcrw.ncu-rep --launches gpurun_out/${T}_launches.csv --launches gpurun_out/${T}_c4_launches.csv \
  > gpurun_out/${T}_ncu_summary.md 2>&1
python scripts/ncu_lines.py /tmp/reps/${T}_fwd.ncu-rep > gpurun_out/${T}_fwd_lines.txt 2>&1
python scripts/ncu_lines.py /tmp/reps/${T}_adj.ncu-rep > gpurun_out/${T}_adj_lines.txt 2>&1
python scripts/ncu_opcodes.py /tmp/reps/${T}_fwd.ncu-rep > gpurun_out/${T}_fwd_opcodes.txt 2>&1
python scripts/ncu_traffic.py fwd_kernel /tmp/reps/${T}_fwd.ncu-rep adj_kernel /tmp/reps/${T}_adj.ncu-rep \
  --config thomas:100:1000:10000 --tag $T > gpurun_out/${T}_traffic.txt 2>&1
cp profiles/traffic.json gpurun_out/${T}_traffic.json
ncu -i /tmp/reps/${T}_node_eval.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for k in h:
    if 'tensor' in k or 'dmma' in k.lower() or 'fp64' in k: print(k, v[h.index(k)])
" > gpurun_out/${T}_node_eval_tensor.txt 2>&1
rm -rf /tmp/reps
tail -c 1500 gpurun_out/${T}_bench.json; tail -3 gpurun_out/${T}_bench.err
ls -la gpurun_out
