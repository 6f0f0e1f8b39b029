set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_p2p.py tests/test_gpu_rows.py -q -m gpu -x -k "launch_configuration or persistent or p2p or row_slabs_match or c1_parity" > gpurun_out/pt29.log 2>&1; echo pt=$?; tail -2 gpurun_out/pt29.log
bash scripts/gpu_sanitize.sh
