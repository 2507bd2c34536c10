timeout 1500 python -m pytest tests/test_gpu_parity_paths.py -k "large or gather" -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02f.log 2>&1
tail -3 gpurun_out/pytest_gpu_r02f.log
timeout 900 python tools/schur_phases.py 24 > gpurun_out/schur_phases5.txt 2>&1
grep n_c gpurun_out/schur_phases5.txt | tail -4
