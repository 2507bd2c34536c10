# P3 panel sweeps (PDIPC_SCHUR_KPW / _KPW0 / _KTAIL / _WU / _SPLIT) at C3 n_c ~ 3000
for v in 100000 0 40 60 80 100; do
  PDIPC_SCHUR_SPLIT=$v timeout 600 python tools/schur_phases.py 24 > gpurun_out/kw.txt 2>&1
  echo "split_min $v: $(grep 'n_c  3001' gpurun_out/kw.txt | tail -1 | awk '{print $9, $10}')"
done
