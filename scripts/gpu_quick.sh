# GPU check: full GPU test suite (incl. the C3 golden) + 1-GPU bench line
set -x
timeout 2000 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_iter.log 2>&1; echo pytest_rc=$?
tail -n 3 gpurun_out/pytest_gpu_iter.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_iter.log').read().strip().splitlines()[-1]); r=d['roofline']; k=d['kernels']
print(round(d['value']/1e9,2), 'G ev_us', round(r['avg_launch_us_events'],1), 'gt_us', round(r['avg_launch_us_globaltimer'],1), 'frac', round(r['frac'],3), 'tail', k['tail_of_sr_iter']['avg_us'], d['iterations_per_step'], d['clocks']['sm_mhz'])"
