# Round-2 profiling pass (run on the GPU box from the repo root; outputs in gpurun_out/): the ncu
# launch list of two timed C4 steps (8 sequences: kernel SHARES are what matters, the launch list
# is serialised and cold-cache), an ncu --set full capture of the main kernels (graph replay off so
# ncu sees individual launches) and its summary, the C5 sweep.
set -x
timeout 1500 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c4.csv python bench.py --seqs 8 --steps 2 --warmup 1 --no-extras \
    --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_c4.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c4.csv > gpurun_out/launches_c4_summary.txt 2>&1
PDIPC_NO_GRAPH=1 timeout 1800 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" \
    -k regex:"k_local_step|k_schur_coop|k_forward_solve|k_backward_solve|k_pair_derivs|k_gather_elastic|k_narrow|k_accd|k_ls_round" \
    -c 14 -o gpurun_out/full_c4 python bench.py --seqs 8 --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-e2e \
    > gpurun_out/ncu_full_c4.log 2>&1
python tools/ncu_summary.py gpurun_out/full_c4.ncu-rep --traffic-json gpurun_out/ncu_traffic.json > gpurun_out/ncu_full_c4_summary.txt 2>&1
timeout 1500 python tools/c5_sweep.py 10k 50k 100k 300k 1M 2M > gpurun_out/c5_sweep.txt 2>&1
for f in gpurun_out/launches_c4_summary.txt gpurun_out/ncu_full_c4_summary.txt gpurun_out/c5_sweep.txt; do tail -n 3 $f; done
