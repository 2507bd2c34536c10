timeout 1500 python -m pytest tests/test_gpu_parity_paths.py -k "gather or native_c3" -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02d.log 2>&1
tail -5 gpurun_out/pytest_gpu_r02d.log
timeout 600 python tools/backend_ablation.py > gpurun_out/backend_ablation.txt 2>&1
cat gpurun_out/backend_ablation.txt
timeout 900 python tools/schur_phases.py 24 > gpurun_out/schur_phases2.txt 2>&1
tail -8 gpurun_out/schur_phases2.txt
