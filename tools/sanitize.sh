# compute-sanitizer over the C1 run, one tool per invocation (outputs in gpurun_out/)
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_c1.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.txt >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
