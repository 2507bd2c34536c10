# One profiling pass of the round (run on the GPU box from the repo root; outputs in gpurun_out/):
# the bench line, the ncu launch list of two timed C2 frames, an ncu --set full capture of the
# main kernels (graph replay off so ncu sees individual launches), the C5 sweep and the C3 probe.
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --c5 "" \
    > gpurun_out/ncu_launch.log 2>&1
PDIPC_NO_GRAPH=1 timeout 1200 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" \
    -k regex:"k_local_step|k_schur_coop|k_forward_solve|k_backward_solve|k_pair_derivs|k_gather_elastic|k_narrow|k_accd|k_ls_round" \
    -c 12 -o gpurun_out/full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --c5 "" \
    > gpurun_out/ncu_full.log 2>&1
timeout 600 python tools/c5_sweep.py 300k 1M > gpurun_out/c5_sweep.txt 2>&1
timeout 900 python tools/c3_probe.py 60 > gpurun_out/c3_probe.txt 2>&1
