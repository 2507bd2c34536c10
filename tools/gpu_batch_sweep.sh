# C4 step vs Schur systems per launch (PDIPC_SCHUR_BATCH)
for k in 2 3 4 1; do
  PDIPC_SCHUR_BATCH=$k timeout 900 python bench.py --steps 6 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/bs_$k.json 2> gpurun_out/bs_$k.err
  echo "systems per launch $k: $(python -c "import json;d=json.loads(open('gpurun_out/bs_$k.json').read().strip().splitlines()[-1]);print(round(d['value'],2), round(d['ms_per_step'],1))")"
done
