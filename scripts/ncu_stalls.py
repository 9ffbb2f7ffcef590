"""Summarise an ncu report: key metrics + top stalled SASS lines with their stall reasons.
Usage: python scripts/ncu_stalls.py report.ncu-rep [topN]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum"]
for i, x in enumerate(h):
    if x in keys:
        print(f"{x:70s} {v[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
ia, isrc = hh.index("Address"), hh.index("Source")
iss = hh.index("Warp Stall Sampling (All Samples)")
iex = hh.index("Instructions Executed")
stall_cols = [i for i, x in enumerate(hh) if x.startswith("stall_") or "Stall" in x and "Sampling" not in x]
body = rows[2:]
tot = sum(int(r[iss] or 0) for r in body)
print("total stall samples", tot)
for r in sorted(body, key=lambda r: -int(r[iss] or 0))[:top]:
    print(f"{r[ia][-5:]} {r[iss]:>6} ex={r[iex]:>7}  {r[isrc][:80]}")
