# one GPU call: ncu launch list + full capture of the iteration kernel, then the bench lines
set -x
TAG=${TAG:-r1} LAUNCHES=1 bash scripts/profile.sh
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$?
tail -c 3000 gpurun_out/bench_full.log; tail -c 1500 gpurun_out/bench_ref.log
