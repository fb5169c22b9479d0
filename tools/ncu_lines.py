"""Per-source-line totals (warp-stall samples, executed instructions) from an ncu report:
  python tools/ncu_lines.py gpurun_out/prof.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, agg = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        n = int(r[hdr.index("Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    agg.append((s, n, f"{fname}:{r[0]}", r[1][:100]))
ts = sum(a[0] for a in agg) or 1
ti = sum(a[1] for a in agg) or 1
print(f"# samples {ts}, warp instructions {ti}")
for s, n, loc, src in sorted(agg, reverse=True)[:top]:
    print(f"{100 * s / ts:5.1f}% stall  {100 * n / ti:5.1f}% inst  {loc:22s} {src}")
