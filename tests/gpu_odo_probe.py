"""GPU probe: odometry chain on embedded grids, several n/chunk combinations."""
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2203_00459_b200 as fb
dev = torch.device("cuda:0")
for n, count, chunk in [(65, 8, 0), (255, 8, 3), (65, 4, 0), (65, 3, 0), (65, 8, 3)]:
    spec = fb.synth_spec(2, n=n, delta=0.5 * 256 / n)
    cfg = fb.MatchConfig.for_grid(n, spec.delta, 360, t_theta=2.0, t_xy=1.0)
    f, g, mf, mg, _ = fb.synth_pairs_host(spec, 40, (count + 1) // 2)
    scans = np.stack([x for p in zip(f, g) for x in p])[:count]
    masks = np.stack([x for p in zip(mf, mg) for x in p])[:count]
    S = torch.from_numpy(scans).to(dev); M = torch.from_numpy(masks).to(dev)
    m = fb.Matcher(cfg, max_batch=count - 1, chunk=chunk)
    try:
        out = m.odometry(S, M, delta=spec.delta)
        torch.cuda.synchronize()
        print(n, count, chunk, "ok", fb.decode_results(out)["status"], flush=True)
        ts = torch.zeros((count - 1, cfg.n_theta), dtype=torch.float64, device=dev)
        xs = torch.zeros((count - 1, n, n), dtype=torch.float32, device=dev)
        out = m.odometry(S, M, delta=spec.delta, theta_surface=ts, xy_surface=xs)
        torch.cuda.synchronize()
        print(n, count, chunk, "surf ok", flush=True)
        bad = scans.copy(); bad[2, 5, 5] = np.inf
        out = m.odometry(torch.from_numpy(bad).to(dev), M, delta=spec.delta)
        torch.cuda.synchronize()
        print(n, count, chunk, "inf ok", fb.decode_results(out)["status"], flush=True)
    except Exception as e:
        print(n, count, chunk, "FAIL", repr(e)[:200], flush=True)
        break
