timeout 900 python tools/schur_phases.py 24 > gpurun_out/schur_phases.txt 2>&1
cat gpurun_out/schur_phases.txt | tail -15
