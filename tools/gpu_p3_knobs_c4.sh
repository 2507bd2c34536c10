# C4 (4 systems per launch) vs the P3 half-panel split threshold (PDIPC_SCHUR_SPLIT: split the panel in
# two halves while >= this many tile columns remain right of it) and the tail panel widths
run() {
  local lab=$1; shift
  env "$@" timeout 900 python bench.py --steps 10 --warmup 4 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/p3_$lab.json 2> gpurun_out/p3_$lab.err
  echo "$lab: $(python -c "import json;d=json.loads(open('gpurun_out/p3_$lab.json').read().strip().splitlines()[-1]);print(round(d['value'],2), round(d['ms_per_step'],1), d['checksum'])")"
}
for v in ${SPLITS:-0 20 30 40}; do run split$v PDIPC_SCHUR_SPLIT=$v; done
