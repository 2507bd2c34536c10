# P3 check: large-system parity tests, then the Schur phase breakdown at C3
timeout 900 python -m pytest tests/test_gpu_parity_paths.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_schur.log 2>&1
tail -3 gpurun_out/pytest_schur.log
timeout 900 python tools/schur_phases.py 24 > gpurun_out/schur_phases.txt 2>&1
grep n_c gpurun_out/schur_phases.txt | tail -3
