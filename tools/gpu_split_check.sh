# work-proportional CTA split of the two Schur systems of a launch: GPU suite, C4 lines
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_split.log 2>&1
tail -3 gpurun_out/pytest_gpu_split.log
timeout 900 python bench.py --steps 10 --warmup 4 --no-extras --no-cpu-baseline > gpurun_out/split_10.json 2> gpurun_out/split_10.err
echo "split 10 steps: $(python -c "import json;d=json.loads(open('gpurun_out/split_10.json').read().strip().splitlines()[-1]);print(round(d['value'],2), round(d['e2e']['value'],2), round(d['ms_per_step'],1), d['checksum'], d['roofline']['frac'])")"
tail -2 gpurun_out/split_10.err
