set -x
timeout 900 python tools/c4_probe.py 8 20 3 > gpurun_out/c4_probe_8.txt 2>&1
timeout 1200 python tools/c4_probe.py 64 20 2 > gpurun_out/c4_probe_64.txt 2>&1
cat gpurun_out/c4_probe_8.txt gpurun_out/c4_probe_64.txt
