# round 2: the full GPU test suite, smoke, the default bench line (with cpu_baseline) and the reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/pytest_full.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_full.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo ref=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_default.log').read().strip().splitlines()[-1]); r=d['roofline']; k=d['kernels']
print('bench', round(d['value']/1e9,2), 'G; ev_us', round(r['avg_launch_us_events'],1), 'frac', round(r['frac'],3), 'tail', k['tail_of_sr_iter']['avg_us'], 'wait', k.get('gridbar_wait',{}).get('avg_us'), d['iterations_per_step'], d['clocks'], 'launches', d['gpu_launches'], 'picard', round(d['picard']['ms_per_time_step'],1))"
tail -c 600 gpurun_out/bench_reference.log
