"""Summarise an ncu --set full capture of the iteration kernel (run here on the .ncu-rep):
key metrics, DRAM bytes vs algorithmic, stall breakdown.  Usage: ncu_summary.py REP [K M n]"""
import collections
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
K, M, n = (int(x) for x in (sys.argv[2:5] if len(sys.argv) > 4 else (9, 5, 2048 * 1024)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]
print("# ncu --set full --clock-control none, k_sr (single-pass PCG-ASSOR-II iteration), C3 2048x1024 K=9, 1 x B200")
for k in keys:
    print(f"{k:80s} {d.get(k, '')}")
unit = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}
u = rows[1][h.index("dram__bytes_read.sum")]
rd = float(d["dram__bytes_read.sum"]) * unit.get(u, 1.0)
wr = float(d["dram__bytes_write.sum"]) * unit.get(rows[1][h.index("dram__bytes_write.sum")], 1.0)
alg = 8.0 * (6 * K * n + 3 * M * n)
print(f"\nDRAM bytes per launch (read+write): {(rd + wr) / 1e6:.1f} MB; algorithmic (odd iteration, "
      f"48 B/DOF vectors + 24 B x M/K coefficients): {alg / 1e6:.1f} MB")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
sh = srows[1]
tot = collections.Counter()
for r in srows[2:]:
    for i, c in enumerate(sh):
        if c.startswith("stall_") and "Not Issued" not in c:
            try:
                tot[c[6:]] += float(r[i])
            except ValueError:
                pass
print("\nwarp stall samples (issued + not issued):")
for k, x in tot.most_common(12):
    print(f"  {k:32s} {int(x)}")
json.dump({"C3:sr_iter": {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                          "duration_us": float(d["gpu__time_duration.sum"])}},
          open("/tmp/ncu_traffic_new.json", "w"), indent=1)
