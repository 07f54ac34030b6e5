# K1-TC CTA-shape variants (scratch builds): C4 full-size matmul time each
for v in "" scratch/var_n6j16 scratch/var_n4j16 scratch/var_n2j32; do
  BBMM_VARIANT=$v timeout 300 python scripts/tc_time.py 2>&1 | tail -1 | sed "s@^@[${v:-default}] @"
done
