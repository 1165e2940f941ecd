#!/bin/bash
# Structured kernels: ncu launch list of one bench step, full captures of fwd2/adj2 (SP), per-line stalls.
mkdir -p gpurun_out /tmp/reps
T=${TAG:-r2c}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 1 \
  --no-e2e --no-cpu-baseline --no-c3 --quiet-clocks > /dev/null 2>&1
for K in fwd adj; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${K}2_kernel" -c 1 \
    -o /tmp/reps/${T}_${K} -f python bench.py --steps 1 --warmup 0 \
    --no-e2e --no-cpu-baseline --no-c3 --quiet-clocks > gpurun_out/${T}_${K}.log 2>&1
  python scripts/ncu_lines.py /tmp/reps/${T}_${K}.ncu-rep > gpurun_out/${T}_${K}_lines.txt 2>&1
done
python scripts/ncu_summary.py /tmp/reps/${T}_fwd.ncu-rep /tmp/reps/${T}_adj.ncu-rep \
  --launches gpurun_out/${T}_launches.csv > gpurun_out/${T}_ncu_summary.md 2>&1
python scripts/ncu_traffic.py fwd_kernel /tmp/reps/${T}_fwd.ncu-rep adj_kernel /tmp/reps/${T}_adj.ncu-rep \
  --config thomas:100:1000:10000 --tag $T > gpurun_out/${T}_traffic.txt 2>&1
cp profiles/traffic.json gpurun_out/${T}_traffic.json
rm -rf /tmp/reps
head -30 gpurun_out/${T}_ncu_summary.md; head -25 gpurun_out/${T}_fwd_lines.txt; head -25 gpurun_out/${T}_adj_lines.txt
