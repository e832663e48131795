# A/B: 160 x 48 Gram tiles for k1 > 128, k2 in (32, 48] (cfg3's bs = 40) at cfg3's n
for T in 0 1; do
  echo "== GCG_GRAM48=$T"
  GCG_GRAM48=$T SHAPES=360x40,400x40,320x40,200x40,600x40 python scripts/gram_big_probe.py 493039 2>&1 | grep -v "^$"
done
GCG_GRAM48=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "gram" 2>&1 | tail -1
