"""cuBLAS DGEMM (torch.matmul, float64, FP64 tensor cores) throughput on this GPU: N^3 x 2 flops,
best of 5 (burst) and back to back for ~4 s (sustained), CUDA events.  The library FP64 reference
the dense Schur kernel's DMMA rate is compared with (bench.py roofline peak)."""
import json
import sys
import time

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
c = a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    c = a @ b
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
k, t0 = 0, time.time()
e0.record()
while time.time() - t0 < 4.0:
    c = a @ b
    k += 1
    if k % 8 == 0:
        torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
sus = e0.elapsed_time(e1) / k
fl = 2.0 * n ** 3
print(json.dumps({"dgemm_n": n, "burst_tflops": fl / best / 1e9, "sustained_tflops": fl / sus / 1e9,
                  "sustained_runs": k}))
