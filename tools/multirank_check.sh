# correctness of the multi-rank bench path on one GPU: the combined per-sequence checksum of P = 2
# ranks (gloo, device shared) must equal the P = 1 run's
python bench.py --seqs 8 --steps 3 --warmup 1 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/p1.json 2> gpurun_out/p1.err
BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
    bench.py --gpus 2 --seqs 8 --steps 3 --warmup 1 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/p2.json 2> gpurun_out/p2.err
python - <<'PY'
import json
a = json.loads(open("gpurun_out/p1.json").read().strip().splitlines()[-1])
b = json.loads(open("gpurun_out/p2.json").read().strip().splitlines()[-1])
print("P=1 checksum", a["checksum"], "P=2 checksum", b["checksum"], "equal", a["checksum"] == b["checksum"])
print("P=2 per-rank ms", b["per_rank_ms"], "sequences_per_gpu", b["config"]["sequences_per_gpu"])
PY
