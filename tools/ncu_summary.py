"""One-line-per-kernel summary of an ncu --set full report (duration, DRAM bytes,
occupancy, issue, bank conflicts, top stalls). usage: python tools/ncu_summary.py rep [--json out]"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
M = {"dur_us": "gpu__time_duration.sum", "dram_rd": "dram__bytes_read.sum", "dram_wr": "dram__bytes_write.sum",
     "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
     "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "regs": "launch__registers_per_thread", "smem_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
     "grid": "launch__grid_size", "block": "launch__block_size",
     "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
     "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed"}
res = []
for r in rows[2:]:
    d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]}
    for k, m in M.items():
        if m in hdr:
            v = r[hdr.index(m)]
            try:
                d[k] = float(v.replace(",", ""))
            except ValueError:
                d[k] = v
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    d["top_stalls"] = [(s, round(v, 2)) for v, s in sorted(st, reverse=True)[:4]]
    res.append(d)
for d in res:
    mb = (d.get("dram_rd", 0) + d.get("dram_wr", 0))
    unit = "MB"  # ncu raw page reports dram bytes in its own unit column; see rows[1]
    print(f"{d['kernel']:28s} {d.get('dur_us', 0):8.1f}us dram {mb:8.2f} dram% {d.get('dram_pct', 0):5.1f} "
          f"sm% {d.get('sm_pct', 0):5.1f} warps% {d.get('warps_active_pct', 0):5.1f} issue% {d.get('issue_pct', 0):5.1f} "
          f"regs {d.get('regs', 0):.0f} bankconf {d.get('smem_conflicts', 0):.0f} {d['top_stalls']}")
units = {h: rows[1][i] for i, h in enumerate(hdr)}
if "--json" in sys.argv:
    json.dump({"report": rep, "units": {k: units.get(m, "") for k, m in M.items()}, "kernels": res},
              open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
