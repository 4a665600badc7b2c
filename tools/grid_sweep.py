"""Throughput over grid sides (powers of two and the reference's odd sizes), 1024
pairs per call (fewer at N = 1024), masks, graph replay, device inputs. Writes one
JSON object per line. usage (GPU): python tools/grid_sweep.py > profiles/r02/grid_sweep.jsonl"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_00459_b200 as fb  # noqa: E402

for n, nt, b in ((64, 360, 1024), (127, 360, 1024), (128, 360, 1024), (255, 733, 1024), (256, 360, 1024),
                 (256, 733, 1024), (511, 720, 1024), (512, 720, 1024), (1023, 1440, 256), (1024, 1440, 256)):
    cfg = fb.MatchConfig.for_grid(n, 0.4, nt)
    spec = fb.synth_spec(2, n=n, delta=0.4)
    f, g, mf, mg, _ = fb.synth_pairs_device(spec, 0, b)
    m = fb.Matcher(cfg, max_batch=b)
    m.set_graphs(True)
    for _ in range(3):
        m.match_device(f, g, mf, mg, delta=0.4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        m.match_device(f, g, mf, mg, delta=0.4)
    e1.record()
    torch.cuda.synchronize()
    rate = reps * b / (e0.elapsed_time(e1) / 1e3)
    print(json.dumps({"n": n, "n_theta": nt, "pairs": b, "pairs_per_s": round(rate, 1),
                      "path": "radix-16 power of two" if n & (n - 1) == 0 else
                      ("prime-factor 15 x 17" if n == 255 else "Bluestein + embedded translation")}), flush=True)
