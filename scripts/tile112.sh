# A/B: 112-wide Gram / LinComb tiles for k2, d in (96, 112] (cfg4's bs = 100)
for T in ${TS:-0 1}; do
  echo "== GCG_GRAM112=$T GCG_LC112=$T"
  GCG_GRAM112=$T GCG_LC112=$T SHAPES=${SH:-300x100,900x100,500x100} python scripts/gram_big_probe.py 2097152 2>&1 | grep -v "^$"
done
GCG_GRAM112=1 GCG_LC112=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "gram or lincomb" 2>&1 | tail -1
