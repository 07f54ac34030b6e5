mkdir -p gpurun_out
for tool in racecheck memcheck synccheck; do
  NV_COMPUTE_SANITIZER_MAX_RACECHECK_HAZARDS=100000 timeout 1200 compute-sanitizer --tool $tool --print-limit 30 python scripts/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "SUMMARY|Race reported between" gpurun_out/sanitize_$tool.log | sed 's/(const.*//' | sort | uniq -c | head -12
done
