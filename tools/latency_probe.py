"""Dev probe: per-call latency of small batches (device inputs), N = 255/256/512."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2203_00459_b200 as fb  # noqa: E402

for graphs, n, nt in [(gr, n, nt) for gr in (True, False, True) for n, nt in ((255, 733), (256, 360), (512, 720))]:
    cfg = fb.MatchConfig.for_grid(n, 0.4, nt)
    spec = fb.synth_spec(2, n=n, delta=0.4)
    for b in (1, 8):
        f, g, mf, mg, _ = fb.synth_pairs_device(spec, 0, b)
        m = fb.Matcher(cfg, max_batch=b)
        m.set_graphs(graphs)
        out = torch.empty(b * fb.RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
        for _ in range(20):
            m.match_device(f, g, mf, mg, delta=0.4, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 200
        t0 = time.perf_counter()
        e0.record()
        for _ in range(reps):
            m.match_device(f, g, mf, mg, delta=0.4, out=out)
        e1.record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / reps * 1e6
        print(f"graphs={int(graphs)} n={n} batch={b}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us/call (device), {wall:.1f} us/call (host)")
