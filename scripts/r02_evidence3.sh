# Round-2 final evidence (one gpurun call): smoke, GPU tests, bench lines (C4 default = 31-bit k~
# grid at n = 1M, C4 forced 23-bit, reference arm, C1-C3), per-config table, ncu launch list of the
# C4 bench, ncu full capture of the C4 bench kernel (MODE 3) and the residual-bound evidence.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
rm -f gpurun_out/fullsize_parity.jsonl
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 1500 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; tail -c 200 gpurun_out/bench_C4.json
timeout 1500 python bench.py --precision int8exact23 --no-cpu-baseline > gpurun_out/bench_C4_23.json 2> gpurun_out/bench_C4_23.err; tail -c 200 gpurun_out/bench_C4_23.json
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 200 gpurun_out/bench_ref.json
for C in C1 C2 C3; do timeout 900 python bench.py --config $C --no-cpu-baseline > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err; tail -c 150 gpurun_out/bench_$C.json; done
timeout 900 python bench.py --config C2 --kmode onthefly --no-cpu-baseline > gpurun_out/bench_C2_otf.json 2> gpurun_out/bench_C2_otf.err; tail -c 150 gpurun_out/bench_C2_otf.json
timeout 900 python scripts/bench_configs.py C0 C1 C2 C3 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; cut -c1-150 gpurun_out/configs.jsonl
timeout 900 python scripts/solve_residual_bound.py 131072 262144 1000000 > gpurun_out/resbound.jsonl 2> gpurun_out/resbound.err; cat gpurun_out/resbound.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1; tail -1 gpurun_out/launches_bench.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k1tc2_rbf -c 1 -o gpurun_out/k1tc2_C4_m3 python scripts/prof_matmul.py 1000000 2 > gpurun_out/prof_c4m3.log 2>&1; tail -1 gpurun_out/prof_c4m3.log
