set -x
timeout 300 python scripts/sanitize.py 2>&1 | tail -8
bash scripts/gpu_sanitize.sh 2>&1 | tee gpurun_out/sanitize_summary.txt
timeout 600 python scripts/probe_rows1.py 2>&1 | tee gpurun_out/rows1.log
timeout 600 python scripts/probe_slab_sizes.py 2>&1 | tee gpurun_out/slab_sizes.log
