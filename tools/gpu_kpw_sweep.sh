for kw in "10 3.6" "10 3.75" "10 3.9" "12 3.75" "8 3.75" "16 3.5"; do set -- $kw
  PDIPC_SCHUR_KPW=$1 PDIPC_SCHUR_WU=$2 timeout 600 python tools/schur_phases.py 24 > gpurun_out/kw.txt 2>&1
  echo "kpw $1 wu $2: $(grep 'n_c  3001' gpurun_out/kw.txt | tail -1 | awk '{print $9, $10}')"
done
