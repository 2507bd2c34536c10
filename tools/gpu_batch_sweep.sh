# C4 step vs Schur systems per launch (PDIPC_SCHUR_BATCH), work-proportional CTA split
for k in ${KS:-4 6 8}; do
  PDIPC_SCHUR_BATCH=$k timeout 900 python bench.py --steps 10 --warmup 4 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/bs_$k.json 2> gpurun_out/bs_$k.err
  echo "systems per launch $k: $(python -c "import json;d=json.loads(open('gpurun_out/bs_$k.json').read().strip().splitlines()[-1]);print(round(d['value'],2), round(d['ms_per_step'],1), d['checksum'])")"
  tail -1 gpurun_out/bs_$k.err
done
timeout 900 python -m pytest tests/test_gpu_lockstep.py -q -p no:cacheprovider > gpurun_out/pytest_bs.log 2>&1; tail -1 gpurun_out/pytest_bs.log
