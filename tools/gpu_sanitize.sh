mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
done
