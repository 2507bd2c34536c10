# C4 (64 sequences) lockstep timeline of sequence 0's slot: where the batched w_el solve sits
PDIPC_TIMELINE=1 timeout 600 python tools/c4_probe.py 64 20 2 30 > gpurun_out/c4_timeline.txt 2>&1
grep -E "timeline|ms_per" gpurun_out/c4_timeline.txt | cut -c1-1500
bash tools/fp64_peak_check.sh
