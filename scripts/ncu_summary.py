"""Summarise an ncu --set full capture of the iteration kernel (run here on the .ncu-rep): key
metrics, DRAM bytes vs algorithmic, stall breakdown (by reason and by opcode), and the traffic
entry for profiles/ncu_traffic.json.

  ncu_summary.py REP [ITERS K M n]

ITERS = PCG iterations inside the captured launch (the persistent kernel k_srp runs a whole
fixed-iteration solve in one launch: scripts/ncu_target.py); per-iteration numbers are the
launch totals / ITERS, the unit of bench.py's roofline (average of even and odd iterations:
8 (5 K n + 3 M n) bytes, the x update every other iteration)."""
import collections
import csv
import io
import json
import re
import subprocess
import sys

rep = sys.argv[1]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
K, M, n = (int(x) for x in (sys.argv[3:6] if len(sys.argv) > 5 else (9, 5, 2048 * 1024)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]
print(f"# ncu --set full --clock-control none, {d.get('Kernel Name', '?')}, C3 2048x1024 K=9, 1 x B200; "
      f"{iters} PCG iteration(s) in the captured launch")
for k in keys:
    if k in d:
        print(f"{k:80s} {d[k]} {u[h.index(k)]}")
scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0, "ms": 1e3, "us": 1.0, "usecond": 1.0,
         "msecond": 1e3, "nsecond": 1e-3, "ns": 1e-3}
rd = float(d["dram__bytes_read.sum"]) * scale.get(u[h.index("dram__bytes_read.sum")], 1.0)
wr = float(d["dram__bytes_write.sum"]) * scale.get(u[h.index("dram__bytes_write.sum")], 1.0)
dur_us = float(d["gpu__time_duration.sum"]) * scale.get(u[h.index("gpu__time_duration.sum")], 1.0)
alg = 8.0 * (5 * K * n + 3 * M * n)
print(f"\nper PCG iteration: DRAM read+write {(rd + wr) / iters / 1e6:.1f} MB, algorithmic "
      f"8 (5 K n + 3 M n) = {alg / 1e6:.1f} MB (ratio {(rd + wr) / iters / alg:.3f}); "
      f"{dur_us / iters:.1f} us under ncu -> {alg / (dur_us / iters * 1e-6) / 1e9:.0f} GB/s algorithmic")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = [r for r in csv.reader(io.StringIO(src))]
sh = srows[1]
ix = {c: i for i, c in enumerate(sh)}
tot, byop = collections.Counter(), collections.defaultdict(collections.Counter)
for r in srows[2:]:
    if len(r) < len(sh):
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", r[ix["Source"]])
    op = m.group(2) if m else "?"
    for c in sh:
        if c.startswith("stall_") and "Not Issued" not in c:
            try:
                x = float(r[ix[c]])
            except ValueError:
                continue
            tot[c[6:]] += x
            byop[op][c[6:]] += x
allv = sum(tot.values())
print("\nwarp stall samples by reason (issued + not issued):")
for k, x in tot.most_common(12):
    print(f"  {k:32s} {int(x):8d} {100 * x / allv:5.1f}%")
print("\nby opcode (top reasons):")
for op, c in sorted(byop.items(), key=lambda kv: -sum(kv[1].values()))[:10]:
    s = sum(c.values())
    print(f"  {op:8s} {100 * s / allv:5.1f}%  " + ", ".join(f"{k} {int(x)}" for k, x in c.most_common(3)))
json.dump({"C3:sr_iter": {"dram_bytes_per_launch": (rd + wr) / iters, "dram_read": rd / iters,
                          "dram_write": wr / iters, "duration_us": dur_us / iters, "iterations_in_capture": iters,
                          "unit": "one PCG iteration (persistent k_srp launch total / iterations)"}},
          open("/tmp/ncu_traffic_new.json", "w"), indent=1)
