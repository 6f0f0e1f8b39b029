set -x
timeout 2400 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_rows.py tests/test_gpu_parity.py -q -m gpu -k "p2p or row or nccl or persistent or c1_parity" > gpurun_out/pt20.log 2>&1; echo pt=$?; tail -6 gpurun_out/pt20.log
