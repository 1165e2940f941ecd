#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_v2.py tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_group.py tests/test_gpu_group_ipc.py tests/test_gpu_chunk_ops.py -q -x > gpurun_out/inv_pytest.log 2>&1
tail -3 gpurun_out/inv_pytest.log
timeout 300 python scripts/c2_pcr_sweep.py thomas,100,1000 thomas,100,125 thomas,100,16 thomas,20,125 thomas,100,296 thomas,100,297 2>&1
