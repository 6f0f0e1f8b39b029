export GMAF_LAUNCH_MODE=stream SAN_CASE=60,25,2,43 SAN_WORLD=3
PORT=$((29500 + RANDOM % 1000))
for r in 0 1; do timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_rows.py $r $PORT > gpurun_out/san3_$r.log 2>&1 & done
timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_rows.py 2 $PORT > gpurun_out/san3_2.log 2>&1
wait
for r in 0 1 2; do echo "rank $r: $(grep 'ERROR SUMMARY' gpurun_out/san3_$r.log) $(grep -h 'slab' gpurun_out/san3_$r.log)"; grep -m3 "Invalid\|at 0x\|by thread" gpurun_out/san3_$r.log; done
