set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import paper_2312_02999_b200.pd_ipc as P; print(P.lib.pd_ipc_build_info())"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_schur_coop -s 450 -c 2 -o gpurun_out/c3_schur python tools/c3_probe.py 24 > gpurun_out/c3_ncu.log 2>&1
ncu -i gpurun_out/c3_schur.ncu-rep --page details --csv > gpurun_out/c3_schur_details.csv 2>&1
ls -la gpurun_out
