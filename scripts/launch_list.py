"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel totals and
shares of the step: launch_list.py CSV ITERATIONS.  ncu's per-launch times are cold-cache and
serialised, so only the shares are comparable with the bench."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot = collections.OrderedDict()
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", ""))
    unit = r[h.index("Metric Unit")]
    us = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v
    tot[r[ik]] = tot.get(r[ik], 0.0) + us
s = sum(tot.values())
it = int(sys.argv[2]) if len(sys.argv) > 2 else 0
print("# ncu --metrics gpu__time_duration.sum --clock-control none: one C3 step (bench.py --steps 1 --warmup 0), "
      "stream launches; cold-cache, serialised: compare shares")
for k, v in tot.items():
    print(f"{k[:60]:62s} {v:12.1f} us {100 * v / s:6.2f}%")
srp = [v for k, v in tot.items() if "k_srp" in k]
msg = f"total {s / 1e3:.1f} ms"
if srp and it:
    msg += f"; k_srp = all PCG iterations of the solve in one launch: {srp[0] / it:.1f} us per iteration"
print(msg)
