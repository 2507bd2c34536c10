timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_schur_coop -s 450 -c 1 -o gpurun_out/c3_schur_r02 python tools/c3_probe.py 24 > gpurun_out/c3_ncu_r02.log 2>&1
ncu -i gpurun_out/c3_schur_r02.ncu-rep --page source --csv --print-source sass > gpurun_out/c3_schur_src_sass.csv 2>&1
ncu -i gpurun_out/c3_schur_r02.ncu-rep --page source --csv --print-source cuda > gpurun_out/c3_schur_src_cuda.csv 2>&1
ncu -i gpurun_out/c3_schur_r02.ncu-rep --page raw --csv > gpurun_out/c3_schur_raw.csv 2>&1
ls -la gpurun_out/c3_schur*
