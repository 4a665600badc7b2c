"""Compile a .cu with -Xptxas -v and print one line per kernel: name, regs, spills, smem."""
import re
import subprocess
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "paper_2203_00459_b200/csrc/kernels.cu"
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Iinclude",
       "-Ipaper_2203_00459_b200/csrc", "-c", src, "-o", "/dev/null", "-Xptxas", "-v"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
rows = []
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        k = re.search(r"k_([a-z_0-9]+?)(?:ILi(\d+)E)?E", name)
        cur = {"k": (k.group(1) + (f"<{k.group(2)}>" if k and k.group(2) else "")) if k else name}
        rows.append(cur)
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur is not None:
        cur["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and cur is not None:
        cur["regs"] = m.group(1)
for r in rows:
    print(f"{r['k']:28s} regs {r.get('regs','?'):>4s}  spill st/ld {r.get('spill','?')}")
