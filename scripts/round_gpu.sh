# One GPU session: smoke, GPU tests, bench JSON (default: e2e + cpu_baseline), reference arm,
# ncu launch list of the bench command, ncu full capture of K1-TC at the full C4 size.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 1500 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1; tail -2 gpurun_out/launches_bench.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k1tc2_rbf -c 1 -o gpurun_out/k1tc2_1M python scripts/prof_matmul.py 1000000 2 > gpurun_out/prof_full.log 2>&1; tail -2 gpurun_out/prof_full.log
