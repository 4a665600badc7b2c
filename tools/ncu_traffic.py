"""profiles/ncu_traffic.json from an ncu --set full capture of one C4 step:
DRAM bytes (read + write) per launch and per pair for every pipeline kernel.
Pairs per launch come from k_finalize's grid (one CTA per pair).
Also records each kernel's issue-slot, warps-active, DRAM, L1 (LSU data-pipe
wavefronts) and FMA-pipe utilisation (what bench.py's roofline.ncu quotes).
usage: python tools/ncu_traffic.py REP SOURCE_NOTE [PAIRS_PER_LAUNCH] > profiles/ncu_traffic.json"""
import csv
import io
import json
import subprocess
import sys

rep, note = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]


units = rows[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
         "second": 1e6, "": 1}


def col(r, name):
    i = hdr.index(name)
    return float(r[i].replace(",", "")) * SCALE.get(units[i], 1)


recs = []
for r in rows[2:]:
    full = r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]
    k = full.split("<")[0].replace("k_", "", 1)
    if k == "xlat_out" and full.rstrip(">").replace(" ", "").endswith(",2"):
        k = "xlat_win"  # the two-pass K5's window pass (MODE = kOutWin), bench.py's stage name
    for suffix in ("_mb", "_multi"):  # launch-bound / multi-pair instantiations report under the stage name
        if k.endswith(suffix):
            k = k[: -len(suffix)]
    pc = {m: col(r, c) for m, c in (("issue_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                                     ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
                                     ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                                     ("l1_lsu_pct", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
                                     ("fma_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"))}
    recs.append((k, col(r, "dram__bytes_read.sum") + col(r, "dram__bytes_write.sum"),
                 col(r, "gpu__time_duration.sum"), col(r, "launch__grid_size"), pc))
if len(sys.argv) > 3:
    ppl = int(sys.argv[3])
else:
    ppl = next(int(g) for k, _, _, g, _ in recs if k == "finalize")
res = {"source": note, "pairs_per_launch": ppl, "n_xy": 512}
for k, b, us, _, pc in recs:
    res[k] = {"dram_bytes_per_launch": b, "dram_bytes_per_pair": b / ppl, "duration_us": round(us, 3),
              **{m: round(v, 1) for m, v in pc.items()}}
print(json.dumps(res, indent=1))
