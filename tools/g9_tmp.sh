timeout 900 python tools/schur_phases.py 24 > gpurun_out/schur_phases4.txt 2>&1
tail -50 gpurun_out/schur_phases4.txt
