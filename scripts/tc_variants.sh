# K1-TC CTA-shape variants (scratch builds): C4 full-size matmul time each
for v in "" scratch/var_sttmlive; do
  BBMM_VARIANT=$v timeout 300 python scripts/tc_time.py 2>&1 | tail -1 | sed "s@^@[${v:-default}] @"
done
