set -x
timeout 600 python scripts/probe_balance.py > gpurun_out/balance.log 2>&1; cat gpurun_out/balance.log
CFG=C2 timeout 600 python scripts/probe_balance.py > gpurun_out/balance_c2.log 2>&1; cat gpurun_out/balance_c2.log
