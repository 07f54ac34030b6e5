# Final round evidence (one gpurun call): smoke, GPU tests, per-config lines, stored bench,
# bench line + reference arm, launch list.
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 900 python scripts/bench_configs.py C0 C1 C2 C3 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; cut -c1-200 gpurun_out/configs.jsonl
timeout 600 python scripts/bench_stored.py C2 C1 > gpurun_out/stored_bench.jsonl 2> gpurun_out/stored_bench.err; cut -c1-200 gpurun_out/stored_bench.jsonl
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 700 gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 200 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1; tail -1 gpurun_out/launches_bench.log
