mkdir -p gpurun_out
rm -f gpurun_out/fullsize_parity.jsonl
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -s --timeout 800 > gpurun_out/fullsize.log 2>&1; grep '^{' gpurun_out/fullsize.log | cut -c1-600; tail -2 gpurun_out/fullsize.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "stored or Stored" --timeout 800 > gpurun_out/stored_tests.log 2>&1; tail -2 gpurun_out/stored_tests.log
timeout 600 python scripts/bench_stored.py C2 > gpurun_out/stored_bench.jsonl 2> gpurun_out/stored_bench.err; head -1 gpurun_out/stored_bench.jsonl | cut -c1-400; tail -3 gpurun_out/stored_bench.err
