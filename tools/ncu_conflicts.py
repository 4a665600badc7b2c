"""Top CUDA source lines by excess shared-memory wavefronts (bank conflicts).
usage: python tools/ncu_conflicts.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, agg = "?", None, []
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
        ex = int(r[hdr.index("L1 Wavefronts Shared Excessive")])
        tot = int(r[hdr.index("L1 Wavefronts Shared")])
    except Exception:
        continue
    if tot:
        agg.append((ex, tot, f"{fname}:{r[0]}", r[1].strip()[:90]))
agg.sort(reverse=True)
T = sum(a[1] for a in agg)
E = sum(a[0] for a in agg)
print(f"shared wavefronts {T}, excessive {E} ({100*E/max(T,1):.1f}%)")
for ex, tot, ln, src in agg[:top]:
    print(f"{ex:10d} / {tot:10d}  {ln:16s} {src}")
