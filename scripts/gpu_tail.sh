set -x
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tail.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_tail.log').read().strip().splitlines()[-1]); r=d['roofline']; k=d['kernels']; n=k['sr_iter']['launches']
print(round(d['value']/1e9,2), 'G ev_us', round(r['avg_launch_us_events'],1), 'gt_us', round(r['avg_launch_us_globaltimer'],1), 'tail', k['tail_of_sr_iter']['avg_us'], d['iterations_per_step'], d['clocks']['sm_mhz'])"
