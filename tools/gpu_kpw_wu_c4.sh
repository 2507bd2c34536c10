# C4 (4 Schur systems per launch, proportional split) vs the P3 panel width and update coefficient
run() {  # $1 label, rest: env assignments
  local lab=$1; shift
  env "$@" timeout 900 python bench.py --steps 10 --warmup 4 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/kw_$lab.json 2> gpurun_out/kw_$lab.err
  echo "$lab: $(python -c "import json;d=json.loads(open('gpurun_out/kw_$lab.json').read().strip().splitlines()[-1]);print(round(d['value'],2), round(d['ms_per_step'],1), d['checksum'])")"
}
run kpw8 PDIPC_SCHUR_KPW=8
run kpw12 PDIPC_SCHUR_KPW=12
run wu3.0 PDIPC_SCHUR_WU=3.0
run wu4.0 PDIPC_SCHUR_WU=4.0
run kpw6 PDIPC_SCHUR_KPW=6
