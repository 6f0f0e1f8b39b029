# GPU correctness: smoke + parity tests (+ optional bench)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
if [ -n "$RUN_BENCH" ]; then timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench_rc=$?; fi
for f in gpurun_out/smoke.log gpurun_out/pytest_gpu.log gpurun_out/bench.log; do [ -f $f ] && { echo "== $f"; tail -n 40 $f | cut -c1-3000; }; done
