# A/B: per-iteration time of baseline builds (abA, abB, ...) vs the working tree, then the GPU suite
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python scripts/probe_ab.py /root/repo/abA /root/repo 2>&1 | tee gpurun_out/ab.log
[ -n "$PYT" ] && timeout 2400 python -m pytest tests -q -m gpu -x $PYT > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
