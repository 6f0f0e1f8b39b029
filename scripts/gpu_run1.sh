set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not c3_full" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench1.log 2>&1; echo bench_rc=$?
for f in gpurun_out/smoke.log gpurun_out/pytest_gpu.log gpurun_out/bench1.log; do echo "== $f"; tail -n 30 $f; done
