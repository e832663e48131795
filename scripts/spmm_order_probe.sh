for O in 0 1; do for V in 4 2; do echo -n "ORDER=$O VEC=$V: "; GCG_SPMM_WIN=0 GCG_SPMM_ORDER=$O GCG_SPMM_VEC=$V python scripts/spmm_probe.py 2>&1; done; done
GCG_SPMM_ORDER=1 ncu --section MemoryWorkloadAnalysis --section MemoryWorkloadAnalysis_Tables --clock-control none -k regex:spmm_csr -s 3 -c 1 python scripts/spmm_probe.py 2>&1 | grep -i "hit rate\|L1/TEX\|Mem Busy\|Max Bandwidth\|L2 Hit" | head -12
ncu --section MemoryWorkloadAnalysis --clock-control none -k regex:spmm_csr -s 3 -c 1 python scripts/spmm_probe.py 2>&1 | grep -i "hit rate\|Mem Busy\|Max Bandwidth" | head -8
