# ncu evidence for the persistent iteration kernel at C3 (one GPU): full set + source, 40 iterations
set -x
export GMAF_LAUNCH_MODE=stream
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_srp -c 1 \
  -o gpurun_out/prof_srp python scripts/ncu_target.py 40 > gpurun_out/prof_srp.log 2>&1; echo ncu=$?
tail -3 gpurun_out/prof_srp.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --picard-steps 0 > gpurun_out/launches_bench.log 2>&1; echo launches=$?
ls -la gpurun_out
