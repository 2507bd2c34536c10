timeout 600 python -m pytest tests/test_gpu_region.py tests/test_gpu_f3.py -q -p no:cacheprovider > gpurun_out/pytest_region_f3.log 2>&1
tail -2 gpurun_out/pytest_region_f3.log
timeout 900 python tools/f3_cost.py > gpurun_out/f3_cost.txt 2> gpurun_out/f3_cost.err
cat gpurun_out/f3_cost.txt; tail -2 gpurun_out/f3_cost.err
