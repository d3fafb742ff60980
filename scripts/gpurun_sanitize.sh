# compute-sanitizer, one tool at a time, on the four small cases (summaries -> gpurun_out/)
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -8 gpurun_out/sanitize_$tool.txt
done
