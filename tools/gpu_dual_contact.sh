# contact stages of a batched Schur group on two streams: GPU suite, C4 line vs PDIPC_SERIAL_CONTACT=1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_dual.log 2>&1
tail -3 gpurun_out/pytest_gpu_dual.log
for v in 0 1; do
  PDIPC_SERIAL_CONTACT=$v timeout 900 python bench.py --steps 10 --warmup 4 --no-extras --no-cpu-baseline > gpurun_out/dual_$v.json 2> gpurun_out/dual_$v.err
  echo "serial_contact $v: $(python -c "import json;d=json.loads(open('gpurun_out/dual_$v.json').read().strip().splitlines()[-1]);print(round(d['value'],2), round(d['e2e']['value'],2), round(d['ms_per_step'],1), d['checksum'])")"
  tail -2 gpurun_out/dual_$v.err
done
