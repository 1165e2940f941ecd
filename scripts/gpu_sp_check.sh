mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_structured.py -x -q --timeout 120 > gpurun_out/sp1.log 2>&1; echo "rc=$?" >> gpurun_out/sp1.log
timeout 900 python -m pytest tests/test_gpu_v2.py tests/test_gpu_headline.py -x -q --timeout 300 -k "mds" > gpurun_out/sp2.log 2>&1; echo "rc=$?" >> gpurun_out/sp2.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/sp_bench.json 2> gpurun_out/sp_bench.err; echo "rc=$?" >> gpurun_out/sp_bench.err
tail -15 gpurun_out/sp1.log; tail -5 gpurun_out/sp2.log; head -c 1500 gpurun_out/sp_bench.json; tail -3 gpurun_out/sp_bench.err
