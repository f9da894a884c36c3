"""Summarise an ncu report's source page (cuda,sass view): stall reasons and the hottest CUDA source lines.

usage: python scripts/ncu_hot.py report.ncu-rep kernel-regex [top] [column]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
col = sys.argv[4] if len(sys.argv) > 4 else "Warp Stall Sampling (All Samples)"  # e.g. "Instructions Executed"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = "?"
hdr = None
per_line = collections.Counter()
stalls = collections.Counter()
src = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r) if h not in src}
        hdr = {}
        for i, h in enumerate(r):
            hdr.setdefault(h, i)
        continue
    if hdr is None or r[0] == "" or not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    src[key] = r[1].strip()[:100]
    try:
        per_line[key] += float(r[hdr[col]] or 0)
    except (ValueError, KeyError):
        pass
    for h, i in hdr.items():
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                stalls[h] += float(r[i] or 0)
            except ValueError:
                pass
T = sum(stalls.values()) or 1
print("stalls:", ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in stalls.most_common(9)))
S = sum(per_line.values()) or 1
for (f, ln), v in per_line.most_common(top):
    print(f"{100 * v / S:5.1f}%  {f}:{ln:<5} {src[(f, ln)]}")
