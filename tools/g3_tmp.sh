set -x
timeout 2400 python -m pytest tests/test_gpu_lockstep.py tests/test_gpu_parity.py tests/test_gpu_parity_paths.py -m gpu -q --durations=0 -p no:cacheprovider > gpurun_out/pytest_gpu_r02b.log 2>&1
tail -60 gpurun_out/pytest_gpu_r02b.log
