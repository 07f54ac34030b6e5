# correctness + C4 full-size timing of the K1-TC kernel
timeout 300 python scripts/tc_check.py 2>&1 | tail -8
timeout 300 python scripts/tc_time.py 2>&1 | tail -1
