mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
timeout 300 python scripts/diag_stored2.py 2>&1 | head -8
timeout 600 python scripts/bench_stored.py C2 C1 > gpurun_out/stored_bench.jsonl 2> gpurun_out/stored_bench.err; cat gpurun_out/stored_bench.jsonl; tail -3 gpurun_out/stored_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2tc_stored -s 1 -c 1 -o gpurun_out/k2tc_C2 python scripts/prof_matmul.py 45730 2 C2 stored > gpurun_out/k2tc_ncu.log 2>&1; tail -2 gpurun_out/k2tc_ncu.log
