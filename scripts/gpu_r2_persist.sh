# round 2: persistent iteration kernel -- smoke, parity subset, C3 bench and slab sizes (persistent vs per-launch)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "persistent or c1_parity or fixed_iterates or warm_start or errors or zero or minimum or c2_parity or many_conditions or closed_forms or ragged" > gpurun_out/pt1.log 2>&1; echo pt1=$?
tail -5 gpurun_out/pt1.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p.log 2>&1; echo bp=$?
GMAF_PERSIST=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_np.log 2>&1; echo bnp=$?
timeout 600 python scripts/probe_slab_sizes.py > gpurun_out/slab_p.log 2>&1
GMAF_PERSIST=0 timeout 600 python scripts/probe_slab_sizes.py > gpurun_out/slab_np.log 2>&1
for f in smoke slab_p slab_np; do echo == $f; tail -6 gpurun_out/$f.log; done
for f in bench_p bench_np; do python -c "
import json,sys; d=json.loads(open('gpurun_out/$f.log').read().strip().splitlines()[-1]); r=d['roofline']; k=d['kernels']
print('$f', round(d['value']/1e9,2), 'G; ev_us', round(r['avg_launch_us_events'],1), 'gt_us', round(r['avg_launch_us_globaltimer'],1), 'frac', round(r['frac'],3), 'tail', k['tail_of_sr_iter']['avg_us'], d['iterations_per_step'], d['clocks'])" || tail -20 gpurun_out/$f.log; done
