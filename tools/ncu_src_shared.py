"""Per-SASS-instruction shared-memory wavefronts of one kernel from an ncu report
(source page): usage ncu_src_shared.py rep kernel_regex [top]. Dev tool."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Address" in r)
ix = {k: i for i, k in enumerate(hdr)}
data = [r for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]


def f(r, k):
    try:
        return float(r[ix[k]])
    except ValueError:
        return 0.0


W, X = "L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive"
print("instructions", len(data), "shared wavefronts", sum(f(r, W) for r in data), "excessive", sum(f(r, X) for r in data))
for r in sorted(data, key=lambda r: -f(r, X))[:top]:
    print(r[ix["Address"]][-5:], r[ix["Source"]].strip()[:56].ljust(56), int(f(r, W)), int(f(r, X)))
