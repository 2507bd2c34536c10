set -x
python -c "import paper_2312_02999_b200.pd_ipc as P; print(P.build_info())"
timeout 2400 python -m pytest tests/test_gpu_parity_paths.py tests/test_gpu_parity.py -m gpu -q --durations=0 -p no:cacheprovider > gpurun_out/pytest_gpu_r02a.log 2>&1
tail -40 gpurun_out/pytest_gpu_r02a.log
