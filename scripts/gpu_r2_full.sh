# round 2: bench + slab-size probe (persistent default), barrier-free timing experiment, full GPU test suite
set -x
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p.log 2>&1; echo bp=$?
python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_p.log').read().strip().splitlines()[-1]); r=d['roofline']; k=d['kernels']
print('bench_p', round(d['value']/1e9,2), 'G; ev_us', round(r['avg_launch_us_events'],1), 'gt_us', round(r['avg_launch_us_globaltimer'],1), 'frac', round(r['frac'],3), 'tail', k['tail_of_sr_iter']['avg_us'], 'wait', k.get('gridbar_wait',{}).get('avg_us'), d['iterations_per_step'], d['clocks'])" || tail -20 gpurun_out/bench_p.log
bash scripts/gpu_r2_nobar.sh
timeout 3000 python -m pytest tests -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_full.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_full.log
