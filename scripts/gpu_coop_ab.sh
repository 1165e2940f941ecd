#!/bin/bash
# A/B of the cooperative consumer: parity of the v2 kernels, then C2 Thomas at 1000 and 125 lanes per GPU.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_v2.py tests/test_gpu_headline.py tests/test_gpu_group.py -q -x > gpurun_out/coop_pytest.log 2>&1
tail -3 gpurun_out/coop_pytest.log
for v in base coop0; do
  lib=""; [ "$v" != base ] && lib="variants/$v.so"
  CKO_LIB_PATH=$lib timeout 300 python scripts/c2_pcr_sweep.py thomas,100,1000 thomas,100,125 thomas,100,16 thomas,20,125 2>&1 | sed "s/^/$v /"
done
