# compute-sanitizer over the two-rank row-slab run: each rank its own top-level process under
# its own sanitizer (so both are instrumented for certain)
export GMAF_LAUNCH_MODE=stream
for tool in memcheck initcheck synccheck; do
  PORT=$((29500 + RANDOM % 1000))
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_rows.py 0 $PORT > gpurun_out/san_rows_${tool}_0.log 2>&1 &
  P0=$!
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_rows.py 1 $PORT > gpurun_out/san_rows_${tool}_1.log 2>&1
  R1=$?
  wait $P0; R0=$?
  for r in 0 1; do echo "$tool rank $r rc=$([ $r = 0 ] && echo $R0 || echo $R1) $(grep 'ERROR SUMMARY' gpurun_out/san_rows_${tool}_$r.log) $(grep -h 'slab' gpurun_out/san_rows_${tool}_$r.log)"; done
done
