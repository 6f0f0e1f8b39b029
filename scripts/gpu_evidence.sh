# Evidence run on one B200: smoke + its launch list, ncu of the persistent kernel, the C3 launch
# list, the default bench line and the reference arm (outputs in gpurun_out/, summarised into
# profiles/ by hand)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/pytest_full.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_full.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?; tail -c 3000 gpurun_out/bench.log
export GMAF_LAUNCH_MODE=stream
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_srp -c 1 \
  -o gpurun_out/prof_srp python scripts/ncu_target.py 40 > gpurun_out/prof_srp.log 2>&1; echo ncu=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --picard-steps 0 > gpurun_out/launches.log 2>&1; echo launches=$?
unset GMAF_LAUNCH_MODE
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo ref=$?
timeout 600 python scripts/probe_rows1.py > gpurun_out/rows1.log 2>&1; cat gpurun_out/rows1.log
timeout 600 python scripts/probe_slab_sizes.py > gpurun_out/slab_sizes.log 2>&1; cat gpurun_out/slab_sizes.log
