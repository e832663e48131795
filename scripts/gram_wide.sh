# A/B of the 160 x 128 Gram tile (GCG_GRAM_WIDE=1) at the cfg4/cfg5 deflation shapes
for W in ${WS:-0 1}; do
  echo "GCG_GRAM_WIDE=$W"
  SHAPES=300x100,900x100,500x100,600x200,200x200 GCG_GRAM_WIDE=$W python scripts/gram_big_probe.py 2097152 2>&1 | grep -v "^$"
done
