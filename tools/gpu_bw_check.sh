# one backward-solve launch per batch (column tiles of 8 sequences): GPU suite, C4 bench line
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_bw.log 2>&1
tail -3 gpurun_out/pytest_gpu_bw.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_bw.json 2> gpurun_out/bench_bw.err
python -c "import json;d=json.loads(open('gpurun_out/bench_bw.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['checksum'], d['rooflines']['backward_solve'], d['rooflines']['w_el_forward'])"
tail -3 gpurun_out/bench_bw.err
