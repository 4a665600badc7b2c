"""Dev probe: per-kernel times of one C4 step, independent pairs vs odometry chain."""
import torch
import paper_2203_00459_b200 as fb

cfg, delta, total = fb.baseline_config(4)
spec = fb.synth_spec(4)
f, g, mf, mg, _ = fb.synth_pairs_device(spec, 0, total)
m = fb.Matcher(cfg, max_batch=total)
seq, seqm = torch.cat([f, g[-1:]]), torch.cat([mf, mg[-1:]])
for name, fn in (("pairs", lambda: m.match_device(f, g, mf, mg, delta=delta)),
                 ("chain", lambda: m.odometry(seq, seqm, delta=delta))):
    fn()
    torch.cuda.synchronize()
    m.set_profiling(True)
    fn()
    torch.cuda.synchronize()
    kt = m.kernel_times()
    m.set_profiling(False)
    print(name, round(sum(v[0] for v in kt.values()), 2), {k: round(v[0], 2) for k, v in kt.items()})
