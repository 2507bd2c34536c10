# C4 step (2 Schur systems per launch, 74 CTAs each) vs the P3 update-split coefficient
for u in 3.5 3.0 4.0 2.75; do
  PDIPC_SCHUR_WU=$u timeout 900 python bench.py --steps 6 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/wu_$u.json 2> gpurun_out/wu_$u.err
  echo "wu $u: $(python -c "import json;d=json.loads(open('gpurun_out/wu_$u.json').read().strip().splitlines()[-1]);print(round(d['value'],2), round(d['ms_per_step'],1))")"
done
