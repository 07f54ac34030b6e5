# Round evidence: bench line (with cpu_baseline), reference arm, launch list of the bench command,
# ncu full captures of the on-the-fly kernel at C4 and C3 (one launch each).
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json; tail -2 gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 400 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1; tail -1 gpurun_out/launches_bench.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k1tc2_rbf -c 1 -o gpurun_out/k1tc2_1M python scripts/prof_matmul.py 1000000 2 > gpurun_out/prof_full.log 2>&1; tail -1 gpurun_out/prof_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1tc2_rbf -c 1 -o gpurun_out/k1tc2_C3 python scripts/prof_matmul.py 200000 2 C3 > gpurun_out/prof_c3.log 2>&1; tail -1 gpurun_out/prof_c3.log
