# A/B of an env knob on the 1-GPU bench (C3), no tests
set -x
for e in "$@"; do
timeout 600 env $e python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ab.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1]); r=d['roofline']; k=d['kernels']
print('[$e]', round(d['value']/1e9,2), 'G ev_us', round(r['avg_launch_us_events'],1), 'gt_us', round(r['avg_launch_us_globaltimer'],1), 'frac', round(r['frac'],3), 'tail', k['tail_of_sr_iter']['avg_us'], d['iterations_per_step'], d['clocks']['sm_mhz'])"
done
