set -x
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tail.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_tail.log').read().strip().splitlines()[-1]); k=d['kernels']; n=k['sr_iter']['launches']
print('tail_us', k['tail_of_sr_iter']['avg_us'], 'cycles: red', k['pcg_phase_a']['total_ms']*1e6/n, 'sync', k['pcg_phase_b']['total_ms']*1e6/n, 'stage', k['pcg_init']['total_ms']*1e6/n, 'timing', k['true_residual']['total_ms']*1e6/n, d['clocks']['sm_mhz'])"
