# A/B of the a2 gather on the C5 1M box: internal tet order (sorted by lowest factor position)
# on/off x gather variant (PDIPC_GATHER, k_elastic.cu).  Run on the GPU box from the repo root.
for cfg in "0 0" "0 1" "0 2" "0 3" "1 0" "1 2"; do
    set -- $cfg
    echo "== no_tet_perm=$1 gather=$2"
    PDIPC_NO_TET_PERM=$1 PDIPC_GATHER=$2 timeout 300 python tools/c5_sweep.py 1M
done
