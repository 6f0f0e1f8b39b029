# round 2: new parity tests (K=72 coupled, band storage, max-norm), Picard march, smoke launch list, default bench
set -x
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_picard.py -q -m gpu -k "k72 or band_storage or c1_parity or c2_parity or ragged or random_states or lockstep or picard or march" > gpurun_out/pt_check.log 2>&1; echo pt=$?
tail -5 gpurun_out/pt_check.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1; echo ncu=$?
grep -o '"k_[a-z_]*[^"]*"' gpurun_out/smoke_launches.csv | sort | uniq -c | head -20
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
tail -c 3000 gpurun_out/bench_default.log
