set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rows.py -q -m gpu -x -k "c1_parity or c2_parity or ragged or random or c3_full_size or converged_vs_full or closed_forms or minimum or dedup or band_storage or row_slabs_match or k72" > gpurun_out/pt23.log 2>&1; echo pt=$?; tail -2 gpurun_out/pt23.log
timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --picard-steps 0 > gpurun_out/bench23.log 2>&1; echo bench=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench23.log').read().strip().splitlines()[-1]); k=d['kernels']
print(round(d['value']/1e9,2), {n: (k[n]['avg_us'], k[n]['GBps']) for n in ('assemble','quadrature','thickness_guard','true_residual','sr_init')})"
