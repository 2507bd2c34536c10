# ncu evidence for the C4 step (run on the GPU box from the repo root; outputs in gpurun_out/): the
# launch list of two timed steps (8 sequences: kernel SHARES are what matters -- serialised,
# cold-cache), an ncu --set full capture of the main kernels (graph replay off) and its summary
# with the per-launch DRAM traffic bench.py reports.
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
for f in gpurun_out/launches_c4_summary.txt gpurun_out/ncu_full_c4_summary.txt; do tail -n 5 $f; done
