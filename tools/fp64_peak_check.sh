# whole-GPU FP64 tensor peaks: DMMA micro-benchmark and cuBLAS DGEMM, with SM clocks sampled
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_gpu_peak tools/micro/dmma_gpu_peak.cu
nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active,power.draw --format=csv,noheader -lms 200 > gpurun_out/fp64_clocks.csv &
SMI=$!
/tmp/dmma_gpu_peak > gpurun_out/fp64_gpu_peak.txt 2>&1
python tools/micro/dgemm_torch.py 8192 >> gpurun_out/fp64_gpu_peak.txt 2>&1
kill $SMI
cat gpurun_out/fp64_gpu_peak.txt; sort gpurun_out/fp64_clocks.csv | uniq -c | sort -rn | head -5
