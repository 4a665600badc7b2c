"""Generate tests/golden/*.npz from the reference's OWN code (oracle/_ref).

Run here (the reference tree is present only in the build container):
    python tests/golden/make_golden.py              # small fixtures (inputs stored)
    python tests/golden/make_golden.py --baseline   # BASELINE-size fixtures (inputs regenerated)
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


WIN = 16  # half-width of the stored xy-surface window (the soft-argmax window, matcher.cpp:57-93)


def input_sha(f, g, mf, mg):
    import hashlib
    h = hashlib.sha256()
    for a in (f, g, mf, mg):
        if a is not None:
            h.update(np.ascontiguousarray(a, dtype=np.float32).tobytes())
    return h.hexdigest()


def run_baseline_case(name, cid, pairs, note):
    """BASELINE-size fixtures: the inputs are NOT stored (tens of MB); they are the
    seeded generator's pairs `pairs` of config `cid` (host renderer, byte-identical
    to the GPU tests' inputs; pinned by a SHA-256 per pair). Stored: the reference's
    bins, poses, diagnostics, full theta surface, the xy surface's (2*WIN+1)^2
    window around the reference peak and max|xy surface|."""
    spec = fb.synth_spec(cid)
    cfg, delta, _ = fb.baseline_config(cid)
    oc = oracle.make_config(**{k: (int(v) if isinstance(v, bool) else v) for k, v in cfg.__dict__.items()})
    outs, shas, wins, xmax = [], [], [], []
    for i in pairs:
        f, g, mf, mg, _ = fb.synth_pairs_host(spec, i, 1)
        if not spec.masks:
            mf = mg = None
        shas.append(input_sha(f[0], g[0], None if mf is None else mf[0], None if mg is None else mg[0]))
        r = oracle.scan_match(f[0], g[0], oc, delta, None if mf is None else mf[0], None if mg is None else mg[0],
                              which="ref")
        outs.append(r)
        xs = np.pad(r.xy_surface, WIN)  # window rows/cols clamp to the grid via zero padding
        wins.append(xs[r.xy_row:r.xy_row + 2 * WIN + 1, r.xy_col:r.xy_col + 2 * WIN + 1])
        xmax.append(np.abs(r.xy_surface).max())
    data = dict(config_id=np.int32(cid), pairs=np.array(pairs, dtype=np.int32), input_sha256=np.array(shas),
                masks=np.int32(1 if spec.masks else 0),
                pose=np.array([[r.theta, r.tx, r.ty] for r in outs]),
                diag=np.array([[r.theta_hard, r.theta_peak, r.xy_hard[0], r.xy_hard[1], r.xy_peak] for r in outs]),
                bins=np.array([[r.theta_bin, r.xy_row, r.xy_col] for r in outs], dtype=np.int32),
                theta_surface=np.stack([r.theta_surface for r in outs]),
                xy_window=np.stack(wins), xy_absmax=np.array(xmax), win=np.int32(WIN),
                cfg=np.array([float(getattr(cfg, k)) for k in CFG_KEYS]), delta=np.float64(delta), note=note)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **data)
    print(name, [tuple(int(x) for x in b) for b in data["bins"]])


def main():
    assert oracle.have_ref(), "needs oracle/_ref (build in the container that has /root/reference)"
    if "--baseline" in sys.argv:  # BASELINE-size fixtures only (slow: reference FFTs at N = 512 / 1024)
        run_baseline_case("baseline_c2_n256", 2, [0, 1, 2, 3, 63],
                          "BASELINE config 2 (256^2, 360 bins, masks, T=1), pairs 0-3 and 63")
        run_baseline_case("baseline_c4_n512", 4, [0, 1, 2, 3, 4, 5, 6, 1000, 4095],
                          "BASELINE config 4 (C3/C4 generator, 512^2, 720 bins, masks), pairs 0-6, 1000, 4095")
        run_baseline_case("baseline_c5_n1024", 5, [0, 1, 2, 1023],
                          "BASELINE config 5 (1024^2, 1440 bins, masks, T=0.5), pairs 0-2 and 1023")
        return
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
