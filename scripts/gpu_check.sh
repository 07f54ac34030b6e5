set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -k "not full_size_pivchol" 2>&1 | tail -30
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -3
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --precision fp32acc 2>&1 | tail -3
