# f3 GPU parity, then the full GPU suite and a short C4 bench line
timeout 600 python -m pytest tests/test_gpu_f3.py -q -p no:cacheprovider -x > gpurun_out/pytest_f3.log 2>&1
tail -3 gpurun_out/pytest_f3.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_all.log 2>&1
tail -3 gpurun_out/pytest_gpu_all.log
timeout 900 python bench.py --gpus 1 --steps 10 --warmup 4 --no-extras --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -c 600 gpurun_out/bench_quick.json
