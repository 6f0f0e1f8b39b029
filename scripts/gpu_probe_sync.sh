set -x
for m in rows cond; do
GMAF_LAUNCH_MODE=stream timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sync_$m.csv python scripts/probe_sync.py $m > gpurun_out/sync_$m.log 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/sync_$m.csv")) if len(r)>10]
hdr=rows[0]; ki=hdr.index("Kernel Name"); vi=hdr.index("Metric Value"); ui=hdr.index("Metric Unit")
for r in rows[1:]: print("$m", r[ki][:60], r[vi], r[ui])
PY
done
for m in rows cond; do python scripts/probe_sync.py $m; done
