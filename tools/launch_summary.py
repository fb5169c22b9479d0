"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: launches, total/mean us, share per kernel.
  python tools/launch_summary.py gpurun_out/launches.csv "<command line>" > profiles/<name>.txt"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(r for r in rows if r[0] == "ID")
iN, iM, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows:
    if len(r) == len(hdr) and r[0].isdigit() and r[iM] == "gpu__time_duration.sum":
        v = float(r[iV].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
        us = v / 1000.0 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1000.0)
        tot[r[iN]] += us
        cnt[r[iN]] += 1
S = sum(tot.values())
print(f"# command: {sys.argv[2] if len(sys.argv) > 2 else '?'}")
print("# per-kernel device time (ncu gpu__time_duration.sum, --clock-control none; cold-cache, serialised launches:")
print("# compare SHARES, not absolute times)")
print("# launches     total_us    mean_us   share  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{cnt[k]:10d} {v:12.1f} {v / cnt[k]:10.2f} {100 * v / S:6.2f}%  {k[:110]}")
