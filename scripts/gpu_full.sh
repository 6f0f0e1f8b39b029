set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench_rc=$?
for f in gpurun_out/smoke.log gpurun_out/pytest_gpu.log gpurun_out/bench_full.log; do echo "== $f"; tail -n 15 $f | cut -c1-3000; done
