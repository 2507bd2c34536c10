timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "c1 or c5 or projections or small" > gpurun_out/pytest_c5.log 2>&1; tail -1 gpurun_out/pytest_c5.log
for v in 4 5; do PDIPC_LS_MINB=$v timeout 600 python tools/c5_sweep.py 1M 2M > gpurun_out/c5_$v.txt 2>&1; echo "minb $v"; tail -3 gpurun_out/c5_$v.txt; done
