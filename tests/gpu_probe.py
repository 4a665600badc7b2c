"""Ad-hoc GPU vs oracle probe (prints diffs per stage); not collected by pytest."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
import oracle  # noqa: E402
import paper_2203_00459_b200 as fb  # noqa: E402


def ocfg(cfg):
    return oracle.make_config(**{k: (int(v) if isinstance(v, bool) else v) for k, v in cfg.__dict__.items()})


def probe(cid, count, n_override=None):
    spec = fb.synth_spec(cid)
    cfg, delta, _ = fb.baseline_config(cid)
    if n_override:
        spec.n = n_override
        cfg = fb.MatchConfig.for_grid(n_override, delta, cfg.n_theta, t_theta=cfg.t_theta, t_xy=cfg.t_xy)
    f, g, mf, mg, truth = fb.synth_pairs_host(spec, 0, count)
    dev = torch.device("cuda", 0)
    F, G, MF, MG = (torch.from_numpy(a).to(dev) for a in (f, g, mf, mg))
    m = fb.Matcher(cfg, max_batch=count)
    # stage 1 magnitude
    mag = m.band_magnitude(F * MF).cpu().numpy()
    fm = (f * mf).astype(np.float32)
    n = cfg.n_xy
    for i in range(min(count, 2)):
        ref = oracle.band_magnitude(fm[i].astype(np.float64), cfg.band_lo, cfg.band_hi)[:, n // 2:]
        err = np.abs(mag[i] - ref).max() / np.abs(ref).max()
        print(f"cfg{cid} n={n} pair{i} band-magnitude rel err {err:.3e}")
    ts = torch.zeros((count, cfg.n_theta), dtype=torch.float64, device=dev)
    xs = torch.zeros((count, n, n), dtype=torch.float32, device=dev)
    out = m.match_device(F, G, MF, MG, delta=delta, theta_surface=ts, xy_surface=xs)
    torch.cuda.synchronize()
    res = fb.decode_results(out)
    ts, xs = ts.cpu().numpy(), xs.cpu().numpy()
    oc = ocfg(cfg)
    for i in range(count):
        t0 = time.time()
        r = oracle.scan_match(f[i], g[i], oc, delta, mf[i], mg[i])
        dt = time.time() - t0
        g_ = res[i]
        tsd = np.abs(ts[i] - r.theta_surface).max() / np.abs(r.theta_surface).max()
        xsd = np.abs(xs[i] - r.xy_surface).max() / np.abs(r.xy_surface).max()
        srt = np.sort(r.theta_surface)[::-1]
        print(f"cfg{cid} pair{i}: bins gpu ({g_['theta_bin']},{g_['xy_row']},{g_['xy_col']}) "
              f"ref ({r.theta_bin},{r.xy_row},{r.xy_col}) | dtheta {g_['theta'] - r.theta:.2e} "
              f"dtx {g_['tx'] - r.tx:.2e} dty {g_['ty'] - r.ty:.2e} | surf err th {tsd:.2e} xy {xsd:.2e} "
              f"| th gap {(srt[0] - srt[1]) / srt[0]:.2e} status {g_['status']} | oracle {dt:.2f}s")


if __name__ == "__main__":
    probe(2, 4, n_override=64)
    probe(2, 4, n_override=128)
    probe(1, 1)
    probe(2, 6)
    probe(4, 2)
    probe(5, 1)
