# bench.py's N>1 path (torchrun, 2 ranks) on a ONE-GPU box: both ranks on cuda:0, gloo for the
# host collectives (GMAF_BENCH_SAME_DEVICE=1) -- a plumbing check, not a scaling measurement
set -x
export GMAF_BENCH_SAME_DEVICE=1
for part in rows conditions; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) \
  bench.py --gpus 2 --steps 2 --warmup 3 --config C2 --partition $part > gpurun_out/bench_2rank_$part.log 2>&1; echo rc=$?
tail -c 1200 gpurun_out/bench_2rank_$part.log; echo
done
