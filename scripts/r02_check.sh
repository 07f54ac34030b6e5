mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -s --timeout 800 > gpurun_out/fullsize.log 2>&1; tail -12 gpurun_out/fullsize.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 -x > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
timeout 600 python scripts/bench_stored.py C2 C1 > gpurun_out/stored_bench.jsonl 2> gpurun_out/stored_bench.err; cut -c1-400 gpurun_out/stored_bench.jsonl; tail -3 gpurun_out/stored_bench.err
