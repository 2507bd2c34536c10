# C4 step (2 Schur systems per launch) vs the P3 panel width
for k in 8 12 6; do
  PDIPC_SCHUR_KPW=$k timeout 900 python bench.py --steps 6 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/kp_$k.json 2> gpurun_out/kp_$k.err
  echo "kpw $k: $(python -c "import json;d=json.loads(open('gpurun_out/kp_$k.json').read().strip().splitlines()[-1]);print(round(d['value'],2), round(d['ms_per_step'],1))")"
done
