for w in 4.0 2.6; do
  PDIPC_SCHUR_WU=$w timeout 600 python tools/schur_phases.py 24 > gpurun_out/sp_$w.txt 2>&1
  echo "wu $w: $(grep 'n_c  3001' gpurun_out/sp_$w.txt | tail -1)"; grep -A3 "P3 detail" gpurun_out/sp_$w.txt
done
