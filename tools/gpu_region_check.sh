# backend 4 (prescribed region) parity, then the f1 ablation with it
timeout 600 python -m pytest tests/test_gpu_region.py -q -p no:cacheprovider -x > gpurun_out/pytest_region.log 2>&1
tail -3 gpurun_out/pytest_region.log
timeout 900 python tools/backend_ablation.py > gpurun_out/backend_ablation.txt 2> gpurun_out/backend_ablation.err
tail -c 1500 gpurun_out/backend_ablation.txt; tail -3 gpurun_out/backend_ablation.err
