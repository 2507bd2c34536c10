# C4 step vs the exponent of the Schur CTA-split weights m^p (PDIPC_SCHUR_WEXP), 4 systems per launch
for p in ${PS:-3 2.5 3.5}; do
  PDIPC_SCHUR_WEXP=$p timeout 900 python bench.py --steps 10 --warmup 4 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/we_$p.json 2> gpurun_out/we_$p.err
  echo "wexp $p: $(python -c "import json;d=json.loads(open('gpurun_out/we_$p.json').read().strip().splitlines()[-1]);print(round(d['value'],2), round(d['ms_per_step'],1), d['checksum'])")"
done
