# compute-sanitizer over every kernel family (tools/sanitize_run.py)
for tool in memcheck racecheck synccheck; do
  echo "## $tool"

  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_run.py > gpurun_out/san_$tool.log 2>&1; grep -E "sanitize run ok|ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/san_$tool.log
done
