# quick perf check: gpu tests (rows + p2p + parity subset) + 1-GPU bench lines
set -x
timeout 1500 python -m pytest tests -q -m gpu -x -k "not c3_converged_vs_full" > gpurun_out/pytest_gpu_iter.log 2>&1; echo pytest_rc=$?
tail -n 2 gpurun_out/pytest_gpu_iter.log
run() {
timeout 600 env $1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline $2 > gpurun_out/bench_iter.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_iter.log').read().strip().splitlines()[-1]); r=d['roofline']
print('bench [$1 $2]', round(d['value']/1e9,2), 'G', 'ms/step', round(d['ms_per_step'],1), 'ev_us', round(r['avg_launch_us_events'],1), 'gt_us', round(r['avg_launch_us_globaltimer'],1), 'frac', round(r['frac'],3), d['clocks']['sm_mhz'])"
}
run "X=1" ""
run "X=1" "--partition rows"
run "GMAF_ROWS_SEPARATE=1" "--partition rows"
