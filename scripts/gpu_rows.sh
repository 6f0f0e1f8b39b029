# row-slab sharding: GPU tests + 1-GPU bench lines (plain and rows machinery on a 1-rank slab)
set -x
timeout 900 python -m pytest tests/test_gpu_rows.py tests/test_gpu_p2p.py -q -x > gpurun_out/pytest_rows.log 2>&1; echo rows_rc=$?
tail -n 5 gpurun_out/pytest_rows.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --partition rows > gpurun_out/bench_rows1.log 2>&1; echo bench_rows_rc=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --shard > gpurun_out/bench_cond1.log 2>&1; echo bench_cond_rc=$?
for f in gpurun_out/bench_rows1.log gpurun_out/bench_cond1.log; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(d['value']/1e9,2), 'G', 'ms/step', round(d['ms_per_step'],1), 'ev_us', round(r['avg_launch_us_events'],1), 'gt_us', round(r['avg_launch_us_globaltimer'],1))"; done
