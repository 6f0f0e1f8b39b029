# quick GPU iteration: sync-kernel launch list, all GPU tests but the C3 golden, 1-GPU bench lines
set -x
bash scripts/gpu_probe_sync.sh 2>/dev/null | grep -E "p2p|k_sr<2, 0>|^rows 12|^cond 12" | sort | uniq -c | sort -rn | head -12
timeout 1500 python -m pytest tests -q -m gpu -x -k "not c3_converged_vs_full" > gpurun_out/pytest_gpu_iter.log 2>&1; echo pytest_rc=$?
tail -n 4 gpurun_out/pytest_gpu_iter.log
for a in "" "--partition rows" "--shard"; do
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline $a > gpurun_out/bench_iter.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_iter.log').read().strip().splitlines()[-1]); r=d['roofline']
print('bench [$a]', round(d['value']/1e9,2), 'G', 'ms/step', round(d['ms_per_step'],1), 'ev_us', round(r['avg_launch_us_events'],1), 'gt_us', round(r['avg_launch_us_globaltimer'],1), 'frac', round(r['frac'],3))"
done
