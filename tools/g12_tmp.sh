t0=$(date +%s)
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err
t1=$(date +%s); echo "ours wall $((t1-t0)) s rc" 
tail -3 gpurun_out/bench_r02a.err
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref_r02a.json 2> gpurun_out/bench_ref_r02a.err
t2=$(date +%s); echo "ref wall $((t2-t1)) s"
tail -3 gpurun_out/bench_ref_r02a.err
cat gpurun_out/bench_ref_r02a.json
