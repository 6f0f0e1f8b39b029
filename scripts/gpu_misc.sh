set -x
timeout 600 python bench.py --shard --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_shard.log 2>&1; echo shard_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --shard --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_shard_trun.log 2>&1; echo trun_rc=$?
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo c2_rc=$?
timeout 600 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; echo c1_rc=$?
for f in bench_shard bench_shard_trun bench_c2 bench_c1; do echo "== $f"; tail -c 900 gpurun_out/$f.log; echo; done
