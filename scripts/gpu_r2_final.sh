# round 2 final: full GPU suite, smoke + its launch list, ncu of the persistent kernel, default bench, reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/pytest_full.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_full.log
export GMAF_LAUNCH_MODE=stream
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_srp -c 1 \
  -o gpurun_out/prof_srp_final python scripts/ncu_target.py 40 > gpurun_out/prof_srp_final.log 2>&1; echo ncu=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_final.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --picard-steps 0 > gpurun_out/launches_final.log 2>&1; echo launches=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1; echo smoke_ncu=$?
unset GMAF_LAUNCH_MODE
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_final.log 2>&1; echo ref=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_final.log').read().strip().splitlines()[-1]); r=d['roofline']; k=d['kernels']
print('bench', round(d['value']/1e9,2), 'G; ev_us', round(r['avg_launch_us_events'],1), 'frac', round(r['frac'],3), 'tail', k['tail_of_sr_iter']['avg_us'], 'wait', k.get('gridbar_wait',{}).get('avg_us'), d['iterations_per_step'], d['clocks'], 'launches', d['gpu_launches'], 'picard', round(d['picard']['ms_per_time_step'],1))"
bash scripts/gpu_sanitize.sh
