set -x
timeout 600 python scripts/probe_rows1.py
timeout 1500 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_rows.py -q -m gpu -x > gpurun_out/pt21.log 2>&1; echo pt=$?; tail -2 gpurun_out/pt21.log
