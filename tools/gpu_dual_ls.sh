# CCD / line search of sequence pairs on two streams: GPU suite, C4 line (10 steps; previous 72.67 it/s)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_dualls.log 2>&1
tail -3 gpurun_out/pytest_gpu_dualls.log
timeout 900 python bench.py --steps 10 --warmup 4 --no-extras --no-cpu-baseline > gpurun_out/dualls.json 2> gpurun_out/dualls.err
echo "dual ls: $(python -c "import json;d=json.loads(open('gpurun_out/dualls.json').read().strip().splitlines()[-1]);print(round(d['value'],2), round(d['e2e']['value'],2), round(d['ms_per_step'],1), d['checksum'])")"
tail -2 gpurun_out/dualls.err
