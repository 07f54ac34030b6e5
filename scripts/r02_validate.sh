# Re-entry validation of HEAD: smoke, GPU tests, C4 + C3 bench lines.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
rm -f gpurun_out/fullsize_parity.jsonl
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/gpu_tests.log 2>&1; tail -15 gpurun_out/gpu_tests.log
timeout 900 python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; tail -c 600 gpurun_out/bench_C3.json
timeout 1500 python bench.py --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; tail -c 600 gpurun_out/bench_C4.json
