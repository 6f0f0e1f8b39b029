# final verification: every GPU test, smoke, default bench line, C2 bench line
set -x
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest_rc=$?
tail -n 3 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; cat gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final2.log 2>&1; echo bench_rc=$?
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo bench_c2_rc=$?
for f in gpurun_out/bench_final2.log gpurun_out/bench_c2.log; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(d['value']/1e9,2), 'G', 'ms/step', round(d['ms_per_step'],2), 'frac', round(r['frac'],3), d['iterations_per_step'], d['clocks'])"; done
