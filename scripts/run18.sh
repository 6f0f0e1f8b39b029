set -x
timeout 1500 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_rows.py tests/test_gpu_parity.py -q -m gpu -x -k "p2p or row or nccl or persistent or c1_parity" > gpurun_out/pt18.log 2>&1; echo pt=$?; tail -4 gpurun_out/pt18.log
timeout 600 python scripts/probe_rows1.py
python scripts/probe_ab.py /root/repo/abA /root/repo
