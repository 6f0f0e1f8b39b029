# A/B: per-iteration time of baseline builds (abA, ...) vs the working tree (also with $ENV2 set),
# arrival balance, a GPU test subset
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python scripts/probe_ab.py /root/repo/abA ${ROOTS:-/root/repo} 2>&1 | tee gpurun_out/ab.log
[ -n "$ENV2" ] && env $ENV2 timeout 900 python scripts/probe_ab.py /root/repo 2>&1 | tee -a gpurun_out/ab.log
[ -n "$BAL" ] && env $ENV2 timeout 600 python scripts/probe_balance.py 2>&1 | tee gpurun_out/balance.log
[ -n "$PYT" ] && env $ENV2 timeout 2400 python -m pytest -q -m gpu -x $PYT > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
