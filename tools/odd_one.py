"""Dev helper: one N = 255 (733 bins) matching batch, for ncu captures of the odd-grid kernels."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2203_00459_b200 as fb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 255
cfg = fb.MatchConfig.for_grid(n, 0.4, 733)
spec = fb.synth_spec(2, n=n, delta=0.4)
f, g, mf, mg, _ = fb.synth_pairs_device(spec, 0, 512)
m = fb.Matcher(cfg, max_batch=512)
for _ in range(2):
    m.match_device(f, g, mf, mg, delta=0.4)
torch.cuda.synchronize()
print("done")
