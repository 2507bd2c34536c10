# P3 panel-width sweep (PDIPC_SCHUR_KPW / _KPW0 / _KTAIL / _WU) at C3 n_c ~ 3000
for kw in "10 0" "4 0" "4 4" "4 3" "4 6" "6 4" "2 4"; do set -- $kw
  PDIPC_SCHUR_KPW0=$1 PDIPC_SCHUR_KTAIL=$2 timeout 600 python tools/schur_phases.py 24 > gpurun_out/kw.txt 2>&1
  echo "kpw0 $1 ktail $2: $(grep 'n_c  3001' gpurun_out/kw.txt | tail -1 | awk '{print $9, $10}')"
done
