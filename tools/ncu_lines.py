"""Aggregate ncu warp-stall samples per CUDA source line for one kernel.
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = "?"
hdr = None
agg = []
tot = 0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    try:
        n = int(r[4])
    except Exception:
        continue
    tot += n
    stalls = [(int(r[i]), hdr[i][6:]) for i in range(len(hdr)) if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i] and r[i].isdigit()]
    agg.append((n, f"{fname}:{r[0]}", r[1].strip()[:80], sorted(stalls, reverse=True)[:3]))
agg.sort(reverse=True)
print(f"total samples {tot}")
for n, ln, src, st in agg[:top]:
    print(f"{100*n/max(tot,1):5.1f}% {ln:16s} {src:80s} {[(s, c) for c, s in st if c]}")
