# SpMM column-panel sweep at the wide-k configs (GCG_SPMM_PANEL = max columns per pass,
# GCG_SPMM_ORDER=1: contiguous row ranges per CTA)
for O in 1 0; do
for P in 0 40 20 16; do
  echo "order=$O panel=$P"; GCG_SPMM_ORDER=$O GCG_SPMM_PANEL=$P KB_ONLY=spmm python scripts/kbench_big.py ${CFGS:-4 5} 2>&1 | grep spmm
done
done
