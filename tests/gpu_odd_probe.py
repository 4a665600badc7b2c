"""Dev probe: throughput on the reference's default grid (255, 733 bins) vs 256."""
import time

import torch

import paper_2203_00459_b200 as fb

for n, nt in ((255, 733), (256, 733), (511, 720), (512, 720)):
    cfg = fb.MatchConfig.for_grid(n, 0.4, nt)
    spec = fb.synth_spec(2, n=n, delta=0.4)
    b = 1024
    f, g, mf, mg, _ = fb.synth_pairs_device(spec, 0, b)
    m = fb.Matcher(cfg, max_batch=b)
    for _ in range(2):
        m.match_device(f, g, mf, mg, delta=0.4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        m.match_device(f, g, mf, mg, delta=0.4)
    e1.record()
    torch.cuda.synchronize()
    print(n, nt, round(5 * b / (e0.elapsed_time(e1) / 1e3)), "pairs/s")

# per-kernel split (profiling mode: one lane, events around every launch)
for n, nt in ((255, 733), (256, 733)):
    cfg = fb.MatchConfig.for_grid(n, 0.4, nt)
    spec = fb.synth_spec(2, n=n, delta=0.4)
    f, g, mf, mg, _ = fb.synth_pairs_device(spec, 0, 1024)
    m = fb.Matcher(cfg, max_batch=1024)
    m.match_device(f, g, mf, mg, delta=0.4)
    m.set_profiling(True)
    m.match_device(f, g, mf, mg, delta=0.4)
    torch.cuda.synchronize()
    print(n, {k: round(v[0], 3) for k, v in m.kernel_times().items()})
    m.set_profiling(False)
