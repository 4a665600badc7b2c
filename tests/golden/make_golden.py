"""Generate tests/golden/*.npz from the reference's OWN code (oracle/_ref).

Run here (the reference tree is present only in the build container):
    python tests/golden/make_golden.py
Each fixture holds float32 inputs (so the fp32 GPU path and the fp64 oracle
see identical values), the config, and the reference scan_match outputs:
pose, diagnostics, integer bins, theta surface and translation surface.
Inputs come from the seeded generator (paper_2203_00459_b200 synth) and from
plain uniform-noise grids like the reference's own tests (verify.cpp:18-23).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2203_00459_b200 as fb  # noqa: E402

CFG_KEYS = ("n_theta", "delta_theta", "t_theta", "n_xy", "delta_xy", "t_xy", "band_lo", "band_hi", "n_radius",
            "pad_angle", "softargmax_window", "normalize_scores")


def run_case(name, f, g, mf, mg, cfg, delta, note):
    oc = oracle.make_config(**{k: (int(v) if isinstance(v, bool) else v) for k, v in cfg.__dict__.items()})
    outs = []
    for i in range(f.shape[0]):
        r = oracle.scan_match(f[i], g[i], oc, delta, None if mf is None else mf[i], None if mg is None else mg[i],
                              which="ref")
        outs.append(r)
    n = f.shape[1]
    data = dict(
        f=f.astype(np.float32), g=g.astype(np.float32),
        pose=np.array([[r.theta, r.tx, r.ty] for r in outs]),
        diag=np.array([[r.theta_hard, r.theta_peak, r.xy_hard[0], r.xy_hard[1], r.xy_peak] for r in outs]),
        bins=np.array([[r.theta_bin, r.xy_row, r.xy_col] for r in outs], dtype=np.int32),
        theta_surface=np.stack([r.theta_surface for r in outs]),
        xy_surface=np.stack([r.xy_surface.astype(np.float64 if n <= 128 else np.float32) for r in outs]),
        cfg=np.array([float(getattr(cfg, k)) for k in CFG_KEYS]), delta=np.float64(delta), note=note)
    if mf is not None:
        data["mf"] = mf.astype(np.float32)
        data["mg"] = mg.astype(np.float32)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **data)
    print(name, f.shape, [tuple(int(x) for x in b) for b in data["bins"]])


def main():
    assert oracle.have_ref(), "needs oracle/_ref (build in the container that has /root/reference)"
    # 1) generator pairs at small sizes, masked, C2 conventions
    for n, nt, cnt in ((64, 90, 3), (128, 180, 2), (256, 360, 1)):
        spec = fb.synth_spec(2, n=n, delta=0.5 * 256 / n)
        cfg = fb.MatchConfig.for_grid(n, spec.delta, nt, t_theta=1.0, t_xy=1.0)
        f, g, mf, mg, _ = fb.synth_pairs_host(spec, 100, cnt)
        run_case(f"synth_n{n}", f, g, mf, mg, cfg, spec.delta, "C2-style generator pairs, masks")
    # 2) C1 conventions (unmasked, stock gains) at 256
    spec = fb.synth_spec(1)
    cfg, delta, _ = fb.baseline_config(1)
    f, g, _, _, _ = fb.synth_pairs_host(spec, 0, 1)
    run_case("c1_n256", f, g, None, None, cfg, delta, "BASELINE config 1, pair 0, unmasked")
    # 3) uniform noise grids, integer circular shift (cf. test_spectral.cpp:175-185)
    rng = np.random.default_rng(2203)
    a = rng.random((2, 64, 64)).astype(np.float32)
    b = np.stack([np.roll(a[0], (3, -5), (0, 1)), np.roll(a[1], (-2, 4), (0, 1))])
    cfg = fb.MatchConfig.for_grid(64, 0.4, 64, band_lo=0.15)
    run_case("noise_shift_n64", a, b, None, None, cfg, 0.4, "uniform noise, circular shifts (3,-5), (-2,4)")


if __name__ == "__main__":
    main()
