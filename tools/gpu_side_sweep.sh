# C4 step vs the CTAs of the side-stream (batched w_el) solve (PDIPC_SIDE_CTAS)
for k in 74 148 110 40; do
  PDIPC_SIDE_CTAS=$k timeout 900 python bench.py --steps 6 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/sc_$k.json 2> gpurun_out/sc_$k.err
  echo "side CTAs $k: $(python -c "import json;d=json.loads(open('gpurun_out/sc_$k.json').read().strip().splitlines()[-1]);print(round(d['value'],2), round(d['ms_per_step'],1))")"
done
