# Round-end evidence on one GPU: ncu launch list + full capture of the iteration kernel (C3),
# the default bench line (with the oracle's cpu_baseline), the reference arm, smoke.
set -x
LAUNCHES=1 TAG=final bash scripts/profile.sh > /dev/null 2>&1; echo profile_rc=$?
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -c 600 gpurun_out/bench_final.log; echo; tail -c 400 gpurun_out/bench_ref.log; echo; cat gpurun_out/smoke.log
ls -la gpurun_out
