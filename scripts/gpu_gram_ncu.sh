#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
SHAPES=900x100,100x100 timeout 300 python scripts/gram_big_probe.py 2097152 2>&1 | tail -2
SHAPES=900x100 ncu --set full --clock-control none -k regex:gram_dmma -s 2 -c 1 -o gpurun_out/gram900 \
    python scripts/gram_big_probe.py 2097152 > /dev/null 2>&1; echo "rc=$?"
python scripts/ncu_summary.py gpurun_out/gram900.ncu-rep | head -30
ncu -i gpurun_out/gram900.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for k in ('sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active','launch__grid_size','launch__shared_mem_per_block_dynamic','launch__occupancy_limit_shared_mem','smsp__warps_active.avg.per_cycle_active'):
    if k in h: print(k, v[h.index(k)])
"
SHAPES=100x100 ncu --set full --clock-control none -k regex:gram -s 2 -c 1 -o gpurun_out/gram100 \
    python scripts/gram_big_probe.py 2097152 > /dev/null 2>&1; echo "rc=$?"
python scripts/ncu_summary.py gpurun_out/gram100.ncu-rep | head -30
rm -f gpurun_out/*.ncu-rep
