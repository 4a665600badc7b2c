"""Dev probe: per-kernel device time of one single-pair call (profiling mode)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2203_00459_b200 as fb  # noqa: E402

for n, nt in ((256, 360), (512, 720)):
    cfg = fb.MatchConfig.for_grid(n, 0.4, nt)
    spec = fb.synth_spec(2, n=n, delta=0.4)
    f, g, mf, mg, _ = fb.synth_pairs_device(spec, 0, 1)
    m = fb.Matcher(cfg, max_batch=1)
    m.set_profiling(True)
    for _ in range(5):
        m.match_device(f, g, mf, mg, delta=0.4)
    torch.cuda.synchronize()
    kt = m.kernel_times()
    print(n, round(sum(v[0] for v in kt.values()) * 1e3, 1), "us total;",
          {k: round(v[0] * 1e3, 1) for k, v in kt.items()})
