# sweep the K1-TC warp stagger (cycles) on the C4 full-size matmul
for s in 0 200 350 500 700; do BBMM_TC2_STAGGER=$s timeout 300 python scripts/tc_time.py 2>&1 | tail -1 | sed "s/^/stagger $s: /"; done
