timeout 1500 python -m pytest tests/test_gpu_parity_paths.py tests/test_gpu_parity.py tests/test_gpu_lockstep.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02g.log 2>&1
tail -3 gpurun_out/pytest_gpu_r02g.log
timeout 900 python tools/schur_phases.py 24 > gpurun_out/schur_phases6.txt 2>&1
grep n_c gpurun_out/schur_phases6.txt | tail -4
