import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2203_00459_b200 as fb
for n_cfg in (2, 4):
    cfg, delta, _ = fb.baseline_config(n_cfg)
    f, g, mf, mg, _ = fb.synth_pairs_host(fb.synth_spec(n_cfg), 0, 4)
    dev = torch.device("cuda", 0)
    F, G, MF, MG = (torch.from_numpy(a).to(dev) for a in (f, g, mf, mg))
    m = fb.Matcher(cfg, max_batch=4)
    try:
        out = m.match_device(F, G, MF, MG, delta=delta); torch.cuda.synchronize()
        print("config", n_cfg, "direct ok", fb.decode_results(out)["theta_bin"])
    except Exception as e:
        print("config", n_cfg, "direct FAIL", e); break
