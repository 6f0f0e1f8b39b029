# compute-sanitizer over scripts/sanitize.py (stream launch mode: the tools cannot follow
# kernel nodes of conditional graphs).  Prints per tool: exit code, error summary, and the
# distinct race classes (writer -> reader source lines) racecheck reported.
export GMAF_LAUNCH_MODE=stream
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$? $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/san_$tool.log | head -1) $(grep -c 'sanitize run done' gpurun_out/san_$tool.log)"
done
grep "Race reported between" gpurun_out/san_racecheck.log | sed 's/+0x[0-9a-f]*//g' | sort | uniq -c
