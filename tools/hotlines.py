"""Aggregate ncu stall samples per CUDA source line (source page, cuda,sass view).

usage: python tools/hotlines.py report.ncu-rep kernel_regex [top] [launch_index]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kre}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
agg = collections.Counter()
srcs = {}
cur = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No" or r[0] == "Function Name":
        continue
    if r[0].isdigit() and len(r) > 4 and r[2] == "-":
        try:
            agg[(cur, int(r[0]))] += int(r[4])
            srcs[(cur, int(r[0]))] = r[1].strip()[:100]
        except ValueError:
            pass
tot = sum(agg.values()) or 1
print(f"total samples {tot}")
for k, v in agg.most_common(top):
    print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]:<5d} {srcs[k]}")
