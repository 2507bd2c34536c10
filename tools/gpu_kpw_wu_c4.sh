# C4 (4 Schur systems per launch, proportional split, split threshold 20) vs the P3 update coefficient / panel width
run() {  # $1 label, rest: env assignments
  local lab=$1; shift
  env "$@" timeout 900 python bench.py --steps 10 --warmup 4 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/kw_$lab.json 2> gpurun_out/kw_$lab.err
  echo "$lab: $(python -c "import json;d=json.loads(open('gpurun_out/kw_$lab.json').read().strip().splitlines()[-1]);print(round(d['value'],2), round(d['ms_per_step'],1), d['checksum'])")"
}
run wu3.25 PDIPC_SCHUR_WU=3.25
run wu3.75 PDIPC_SCHUR_WU=3.75
run kpw12 PDIPC_SCHUR_KPW=12
