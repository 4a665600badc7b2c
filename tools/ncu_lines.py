"""Aggregate ncu warp-stall samples per CUDA source line for one kernel.
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top] [inst]  (inst: sort by instructions)"""
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
        ninst = int(r[hdr.index("Instructions Executed")]) if r[hdr.index("Instructions Executed")].isdigit() else 0
    except Exception:
        continue
    tot += n
    itot = globals().setdefault("itot", [0])
    itot[0] += ninst
    stalls = [(int(r[i]), hdr[i][6:]) for i in range(len(hdr)) if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i] and r[i].isdigit()]
    agg.append((n, f"{fname}:{r[0]}", r[1].strip()[:70], sorted(stalls, reverse=True)[:3], ninst))
agg.sort(reverse=True, key=(lambda a: a[4]) if 'inst' in sys.argv[4:] else None)
it = globals().get("itot", [1])[0]
print(f"total samples {tot}, warp instructions {it}")
for n, ln, src, st, ni in agg[:top]:
    print(f"{100*n/max(tot,1):5.1f}% inst {100*ni/max(it,1):5.1f}% {ln:16s} {src:70s} {[(s, c) for c, s in st if c][:2]}")
