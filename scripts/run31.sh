set -x
python scripts/probe_ab.py /root/repo/abA /root/repo
timeout 600 python scripts/probe_balance.py
