"""The parity oracle itself (CPU, no GPU): the C restatement (oracle/liboracle.so)
pinned against the reference's own code — via the golden vectors that
oracle/_ref produced (tests/golden/make_golden.py) and, when the reference tree
is present, live — plus the reference's known-answer properties
(test_spectral.cpp, test_matcher.cpp, verify.cpp)."""
import glob
import math
import os

import numpy as np
import pytest

from conftest import oracle_cfg

GOLDEN = sorted(p for p in glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz"))
                if not os.path.basename(p).startswith("baseline_"))
BASELINE_GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "baseline_*.npz")))
CFG_KEYS = ("n_theta", "delta_theta", "t_theta", "n_xy", "delta_xy", "t_xy", "band_lo", "band_hi", "n_radius",
            "pad_angle", "softargmax_window", "normalize_scores")


def golden_cfg(orc, z):
    vals = dict(zip(CFG_KEYS, z["cfg"]))
    ints = ("n_theta", "n_xy", "n_radius", "pad_angle", "softargmax_window", "normalize_scores")
    return orc.make_config(**{k: (int(v) if k in ints else float(v)) for k, v in vals.items()})


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_restatement_matches_reference_golden(orc, path):
    z = np.load(path)
    cfg = golden_cfg(orc, z)
    for i in range(z["f"].shape[0]):
        mf = z["mf"][i] if "mf" in z else None
        mg = z["mg"][i] if "mg" in z else None
        r = orc.scan_match(z["f"][i], z["g"][i], cfg, float(z["delta"]), mf, mg)
        np.testing.assert_array_equal([r.theta_bin, r.xy_row, r.xy_col], z["bins"][i])
        np.testing.assert_allclose([r.theta, r.tx, r.ty], z["pose"][i], rtol=0, atol=1e-12)
        np.testing.assert_allclose(r.theta_surface, z["theta_surface"][i], rtol=1e-12, atol=0)
        tol = 1e-12 if z["xy_surface"].dtype == np.float64 else 1e-6
        ref = z["xy_surface"][i].astype(np.float64)
        assert np.abs(r.xy_surface - ref).max() <= tol * np.abs(ref).max()


def test_noise_shift_golden_lands_on_exact_lag():
    # roll by (3,-5): content 3 rows down (t_y' = -3 cells), 5 cols left (t_x' = -5)
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "noise_shift_n64.npz"))
    half = (64 - 1) // 2
    assert tuple(z["bins"][0][1:]) == (half - 3, half - 5)
    assert tuple(z["bins"][1][1:]) == (half + 2, half + 4)


def test_next_fast_size(orc):  # test_spectral.cpp:231-240
    L = orc.lib("oracle")
    for n, want in ((1, 1), (7, 7), (11, 12), (13, 14), (121, 125), (509, 512), (2 * 255 - 1, 512),
                    (2 * 256 - 1, 512), (2 * 512 - 1, 1024), (2 * 1024 - 1, 2048)):
        assert L.fo_next_fast_size(n) == want


def direct_xcorr(a, b):
    rows, cols = a.shape
    out = np.zeros_like(a)
    for k in range(rows):
        for l in range(cols):
            out[k, l] = np.sum(a * np.roll(np.roll(b, -(k - rows // 2), 0), -(l - cols // 2), 1))
    return out


def test_xcorr_equals_direct_loop(orc):  # test_spectral.cpp:148-162
    rng = np.random.default_rng(21)
    a, b = rng.random((6, 6)), rng.random((6, 6))
    np.testing.assert_allclose(orc.xcorr(a, b), direct_xcorr(a, b), rtol=1e-9, atol=1e-12)
    a, b = rng.random((9, 5)), rng.random((9, 5))  # odd / non-square, the rotation-stage shapes
    np.testing.assert_allclose(orc.xcorr(a, b), direct_xcorr(a, b), rtol=1e-9, atol=1e-12)


def test_integer_circular_shift_lands_on_lag_bin(orc):  # test_spectral.cpp:175-185
    rng = np.random.default_rng(77)
    a = rng.random((16, 16))
    b = np.roll(a, (3, -5), (0, 1))
    s = orc.xcorr(a, b)
    arg = int(np.argmax(s))
    assert (arg // 16, arg % 16) == (11, 3)


def test_band_magnitude_is_shift_invariant_and_banded(orc):  # test_spectral.cpp:126-132, imageops band
    rng = np.random.default_rng(9)
    g = rng.random((32, 32))
    m = orc.band_magnitude(g, 0.0, 1.0)
    w = 0.5 * (1 - np.cos(2 * np.pi * np.arange(32) / 31))
    ref = np.abs(np.fft.fftshift(np.fft.fft2(g * np.outer(w, w))))
    c = 16
    ii, jj = np.meshgrid(np.arange(32), np.arange(32), indexing="ij")
    rho = np.hypot(ii - c, jj - c) / 16.0
    np.testing.assert_allclose(m, ref * (rho <= 1.0), rtol=1e-10, atol=1e-10)
    m2 = orc.band_magnitude(g, 0.1, 0.5)
    assert np.all(m2[(rho < 0.1) | (rho > 0.5)] == 0.0)


def surface(scores):
    rows, cols = scores.shape
    return np.arange(rows) - rows / 2.0, np.arange(cols) - cols / 2.0


def test_soft_argmax_contracts(orc):  # test_matcher.cpp:105-206
    s = np.zeros((9, 9))
    s[2, 6] = 5.0
    rc, cc = surface(s)
    r, c = orc.soft_argmax(s, rc, cc, 50.0, 2, True)
    assert r == pytest.approx(2 - 4.5, rel=1e-6) and c == pytest.approx(6 - 4.5, rel=1e-6)
    s = np.zeros((1, 7))
    s[0, 2] = s[0, 4] = 1.0
    r, c = orc.soft_argmax(s, [0.0], np.arange(7.0), 200.0, 6, True)
    assert r == 0.0 and c == pytest.approx(3.0, rel=1e-6)
    s = np.ones((5, 5))
    rc, cc = surface(s)
    r, c = orc.soft_argmax(s, rc, cc, 2.0, 16, True)
    assert r == pytest.approx(-0.5, abs=1e-9) and c == pytest.approx(-0.5, abs=1e-9)
    a = np.exp(-0.4 * (np.arange(11) - 5.2) ** 2)[None]
    ra = orc.soft_argmax(a, [0.0], np.arange(11.0), 3.0, 4, True)
    rb = orc.soft_argmax(a * 1000, [0.0], np.arange(11.0), 3.0, 4, True)
    rc_ = orc.soft_argmax(a * 1000, [0.0], np.arange(11.0), 3.0, 4, False)
    assert ra[1] == pytest.approx(rb[1], rel=1e-12) and abs(rc_[1] - ra[1]) > 1e-6


def test_soft_argmax_matches_direct_weighted_mean(orc):  # test_matcher.cpp:143-183
    n = 21
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    s = np.exp(-0.1 * ((i - 9.3) ** 2 + (j - 11.6) ** 2))
    rc, cc = surface(s)
    r, c = orc.soft_argmax(s, rc, cc, 4.0, 5, False)
    pr, pc = np.unravel_index(np.argmax(s), s.shape)
    win = s[max(0, pr - 5):pr + 6, max(0, pc - 5):pc + 6]
    w = np.exp(4.0 * (win - s[pr, pc]))
    rr = rc[max(0, pr - 5):pr + 6][:, None]
    ccw = cc[max(0, pc - 5):pc + 6][None, :]
    assert r == pytest.approx((w * rr).sum() / w.sum(), rel=1e-12)
    assert c == pytest.approx((w * ccw).sum() / w.sum(), rel=1e-12)


def test_config_finalize_and_validate(orc):  # test_matcher.cpp:60-103 (minus the odd-n rule, D1)
    import ctypes as C
    L = orc.lib("oracle")
    cfg = orc.make_config()
    assert L.fo_validate(C.byref(cfg), None, 0) == 0
    d = orc.make_config(n_xy=65, n_theta=100, delta_theta=math.pi / 100, n_radius=0, pad_angle=-1)
    orc.finalize(d)
    assert (d.n_radius, d.pad_angle) == (33, 13)
    t = orc.make_config(n_theta=2, delta_theta=0.01, pad_angle=-1)
    orc.finalize(t)
    assert t.pad_angle == 1
    for kw in (dict(band_lo=0.8), dict(delta_theta=math.pi / 64.0), dict(pad_angle=129),
               dict(softargmax_window=0), dict(t_theta=0.0)):
        bad = orc.make_config(n_xy=65, delta_xy=0.4, n_theta=129, delta_theta=math.pi / 129, n_radius=33,
                              pad_angle=17, band_lo=0.15)
        for k, v in kw.items():
            setattr(bad, k, v)
        assert L.fo_validate(C.byref(bad), None, 0) == 1, kw
    even = orc.make_config(n_xy=64)
    assert L.fo_validate(C.byref(even), None, 0) == 0  # D1: even n accepted


def test_scan_match_rejects_nonfinite_and_bad_masks(orc):  # test_matcher.cpp:362-372
    cfg = orc.make_config(n_xy=64, delta_xy=0.4, n_theta=64, delta_theta=math.pi / 64, n_radius=0,
                          pad_angle=-1, band_lo=0.15)
    orc.finalize(cfg)
    f = np.zeros((64, 64))
    g = np.zeros((64, 64))
    f[3, 3] = np.nan
    with pytest.raises(orc.OracleError):
        orc.scan_match(f, g, cfg, 0.4)
    f[3, 3] = 0.0
    g[1, 1] = np.inf
    with pytest.raises(orc.OracleError):
        orc.scan_match(f, g, cfg, 0.4)
    g[1, 1] = 0.0
    m = np.ones((64, 64))
    m[0, 0] = 1.5
    with pytest.raises(orc.OracleError):
        orc.scan_match(f, g, cfg, 0.4, m, np.ones((64, 64)))


def test_polar_to_cart_spec(orc):
    # a sweep that is constant along range returns that azimuth's value
    n_az, n_rng = 8, 50
    p = np.tile(np.arange(n_az, dtype=np.float64)[:, None], (1, n_rng))
    out = orc.polar_to_cart(p, 1.0, 9, 1.0)
    half = 4
    assert out[half, half + 3] == pytest.approx(0.0)        # +x axis: azimuth 0
    assert out[half - 3, half] == pytest.approx(2.0)        # +y axis: azimuth 2 (of 8)
    assert out[half + 3, half] == pytest.approx(6.0)        # -y axis
    # outside the last range bin: zero
    out2 = orc.polar_to_cart(p[:, :2], 1.0, 9, 1.0)
    assert out2[0, 0] == 0.0


ref_only = pytest.mark.skipif(not os.path.isdir("/root/reference/proj"),
                              reason="reference tree only in the build container")


@ref_only
def test_reference_verify_suites_pass_with_shim(orc):
    fails, report = orc.ref_verify()
    assert fails == 0, report
    assert report.count("[PASS]") == 7


@ref_only
@pytest.mark.parametrize("n,nt", [(65, 129), (64, 90), (128, 180)])
def test_restatement_bit_exact_vs_reference_live(orc, n, nt):
    rng = np.random.default_rng(n)
    f = rng.random((n, n))
    g = np.roll(f, (2, -1), (0, 1)) + 0.01 * rng.random((n, n))
    cfg = orc.make_config(n_xy=n, delta_xy=0.4, n_theta=nt, delta_theta=math.pi / nt, n_radius=0, pad_angle=-1,
                          band_lo=0.15)
    orc.finalize(cfg)
    a = orc.scan_match(f, g, cfg, 0.4)
    b = orc.scan_match(f, g, cfg, 0.4, which="ref")
    assert (a.theta, a.tx, a.ty) == (b.theta, b.tx, b.ty)
    np.testing.assert_array_equal(a.theta_surface, b.theta_surface)
    np.testing.assert_array_equal(a.xy_surface, b.xy_surface)
    for th in (0.0, 0.3, -0.22):
        np.testing.assert_array_equal(orc.rotate_bilinear(f, th), orc.rotate_bilinear(f, th, which="ref"))
    np.testing.assert_array_equal(orc.cart2pol(f, 90, 33, math.pi), orc.cart2pol(f, 90, 33, math.pi, which="ref"))


# ---- exhaustive search (proj/src/oracle.cpp, proj/tests/test_oracle.cpp) ----

def _blobs(n, seed, count=12):
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:n, 0:n].astype(np.float64)
    img = np.zeros((n, n))
    for _ in range(count):
        cy, cx = rng.uniform(0.15 * n, 0.85 * n, 2)
        s = rng.uniform(1.5, 3.0)
        img += rng.uniform(0.3, 1.0) * np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * s * s))
    return img


def test_brute_force_self_match_scores_total_power(orc):  # test_oracle.cpp:96-110
    f = np.random.default_rng(4).random((33, 33))
    r = orc.brute_force(f, f, [-0.2, 0.0, 0.2], 0.4)
    assert (r.theta, r.tx, r.ty) == (0.0, 0.0, 0.0)
    assert r.score == pytest.approx(float((f * f).sum()), rel=1e-9)


def test_brute_force_integer_shift_single_candidate(orc):  # test_oracle.cpp:112-122
    f = _blobs(64, 31)
    g = np.zeros_like(f)
    g[:-3, 5:] = f[3:, :-5]  # content moved -3 rows, +5 cols: world t = (+5, +3) cells
    r = orc.brute_force(f, g, [0.0], 0.4)
    assert r.theta == 0.0
    assert abs(r.tx - 5 * 0.4) < 1e-12 and abs(r.ty - 3 * 0.4) < 1e-12


def test_brute_force_matches_spatial_triple_loop(orc):  # test_oracle.cpp:48-89, 124-134
    n = 12
    rng = np.random.default_rng(7)
    f, g = rng.random((n, n)) - 0.5, rng.random((n, n)) - 0.5
    thetas = [k * 0.1 for k in range(-3, 4)]
    half = (n - 1) // 2
    best = (-1e300, 0.0, 0, 0)
    for th in thetas:
        gr = orc.rotate_bilinear(g, -th)
        for i in range(n):
            for j in range(n):
                oy, ox = i - half, j - half
                r0, r1 = max(0, oy), min(n, n + oy)
                c0, c1 = max(0, -ox), min(n, n - ox)
                acc = float((f[r0:r1, c0:c1] * gr[r0 - oy:r1 - oy, c0 + ox:c1 + ox]).sum())
                if acc > best[0]:
                    best = (acc, th, i, j)
    r = orc.brute_force(f, g, thetas, 0.5)
    assert r.score == pytest.approx(best[0], rel=1e-6)
    assert r.theta == pytest.approx(best[1], abs=1e-12)
    assert (r.xy_row, r.xy_col) == (best[2], best[3])


def test_brute_force_rejects_empty_candidate_list(orc):  # test_oracle.cpp:162-167
    with pytest.raises(orc.OracleError):
        orc.brute_force(np.zeros((8, 8)), np.zeros((8, 8)), [], 0.4)


@ref_only
@pytest.mark.parametrize("n", [33, 64])
def test_brute_force_restatement_bit_exact_vs_reference(orc, n):
    f = _blobs(n, 100 + n)
    rng = np.random.default_rng(n)
    g = np.roll(f, (2, -1), (0, 1)) + 0.05 * rng.random((n, n))
    thetas = np.arange(-6, 7) * 0.05
    a = orc.brute_force(f, g, thetas, 0.4)
    b = orc.brute_force(f, g, thetas, 0.4, which="ref")
    assert (a.theta, a.tx, a.ty, a.score) == (b.theta, b.tx, b.ty, b.score)
    assert (a.theta_index, a.xy_row, a.xy_col) == (b.theta_index, b.xy_row, b.xy_col)


def test_restatement_three_halves_padding_equals_reference_size(orc):
    """The GPU's length-3N/2 circular correlation equals the reference's
    next_fast_size(2N-1) zero-padded one on every kept lag."""
    n = 64
    rng = np.random.default_rng(3)
    f = rng.random((n, n))
    g = np.roll(f, (2, -3), (0, 1)) + 0.1 * rng.random((n, n))
    cfg = orc.make_config(n_xy=n, delta_xy=0.4, n_theta=90, delta_theta=math.pi / 90, n_radius=0, pad_angle=-1,
                          band_lo=0.15)
    orc.finalize(cfg)
    a = orc.estimate_translation_ex(f, g, 0.1, cfg, 0.4, 0, False)
    b = orc.estimate_translation_ex(f, g, 0.1, cfg, 0.4, 3 * n // 2, False)
    assert np.abs(a[2] - b[2]).max() <= 1e-12 * np.abs(a[2]).max()
    assert abs(a[0] - b[0]) < 1e-12 and abs(a[1] - b[1]) < 1e-12


@pytest.mark.parametrize("path", BASELINE_GOLDEN, ids=[os.path.basename(p) for p in BASELINE_GOLDEN])
def test_restatement_matches_baseline_size_golden(orc, path):
    """The fp64 restatement against the reference's own outputs at the BASELINE
    sizes (N = 256 / 512 / 1024; tests/golden/make_golden.py --baseline). Inputs are
    regenerated by the seeded generator (oracle/libsynth_gen.so) and pinned by the
    fixture's SHA-256; the first two pairs of each fixture keep the CPU suite short
    (the GPU test runs them all)."""
    import hashlib
    z = np.load(path)
    cfg = golden_cfg(orc, z)
    delta = float(z["delta"])
    w = int(z["win"])
    for i, p in enumerate(int(x) for x in z["pairs"][:2]):
        f, g, mf, mg, _ = orc.synth_pairs_host(int(z["config_id"]), p, 1)
        if not int(z["masks"]):
            mf = mg = None
        h = hashlib.sha256()
        for a in (f[0], g[0]) + ((mf[0], mg[0]) if mf is not None else ()):
            h.update(a.tobytes())
        assert h.hexdigest() == str(z["input_sha256"][i])
        r = orc.scan_match(f[0], g[0], cfg, delta, None if mf is None else mf[0], None if mg is None else mg[0])
        np.testing.assert_array_equal([r.theta_bin, r.xy_row, r.xy_col], z["bins"][i])
        np.testing.assert_allclose([r.theta, r.tx, r.ty], z["pose"][i], rtol=0, atol=1e-12)
        np.testing.assert_allclose(r.theta_surface, z["theta_surface"][i], rtol=1e-12, atol=0)
        win = np.pad(r.xy_surface, w)[r.xy_row:r.xy_row + 2 * w + 1, r.xy_col:r.xy_col + 2 * w + 1]
        assert np.abs(win - z["xy_window"][i]).max() <= 1e-12 * z["xy_absmax"][i]


# ---------------------------------------------------------------- pins for the rows with no reference code
# SURVEY a20 (polar -> Cartesian, K0) and a21 (phase correlation) have no
# reference implementation; the C restatement is pinned here against
# independent third-party algorithms (scipy.ndimage bilinear, numpy.fft).

def _polar_to_cart_scipy(polar, res, n, delta):
    """K0 spec through scipy.ndimage.map_coordinates(order=1):
    cell (r, c) at x = (c - (n-1)//2) delta, y = -(r - (n-1)//2) delta; azimuth
    bin a centred on 2 pi a / n_az (wrapping), range bin k on (k + 0.5) res,
    range taps outside [0, n_range) read 0. The azimuth wrap and the zero range
    border are made explicit by padding (one wrapped row each side, one zero
    column each side) so one mode='constant' call covers both axes."""
    from scipy import ndimage
    n_az, n_range = polar.shape
    half = (n - 1) // 2
    c, r = np.meshgrid(np.arange(n), np.arange(n))
    x = (c - half) * delta
    y = -(r - half) * delta
    phi = np.mod(np.arctan2(y, x), 2 * np.pi)
    fa = phi * n_az / (2 * np.pi)
    fk = np.hypot(x, y) / res - 0.5
    padded = np.zeros((n_az + 2, n_range + 2))
    padded[1:-1, 1:-1] = polar
    padded[0, 1:-1] = polar[-1]
    padded[-1, 1:-1] = polar[0]
    coords = np.stack([fa + 1.0, fk + 1.0])
    return ndimage.map_coordinates(padded, coords, order=1, mode="constant", cval=0.0, prefilter=False)


@pytest.mark.parametrize("n_az,n_range,res,n,delta", [(400, 3768, 0.0438, 64, 2.0), (37, 120, 0.5, 48, 1.3),
                                                      (400, 300, 0.0438, 96, 0.2)])
def test_polar_to_cart_restatement_equals_scipy_bilinear(orc, n_az, n_range, res, n, delta):
    rng = np.random.default_rng(n_az + n)
    polar = rng.random((n_az, n_range))
    ours = orc.polar_to_cart(polar, res, n, delta)
    ref = _polar_to_cart_scipy(polar, res, n, delta)
    assert np.abs(ours - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
    # the last case runs off the end of the sweep: those cells are exactly zero in both
    assert (ref == 0).any() == ((ours == 0).any())


def _phase_corr_numpy(f, gr, n):
    """Phase correlation on the length-3n/2 grid with numpy.fft:
    X = conj(F) G / |conj(F) G| (0 where 0), c = real(ifft2(X)) (1/M^2 scaling as
    xcorr, spectral.cpp:146-151), centred (fftshift), cropped and flipped like
    matcher.cpp:171-182: s[i, j] = raw[M/2 - (i - half), M/2 + (j - half)]."""
    m = 3 * n // 2
    off = (m - n) // 2
    fp = np.zeros((m, m))
    gp = np.zeros((m, m))
    fp[off:off + n, off:off + n] = f
    gp[off:off + n, off:off + n] = gr
    x = np.conj(np.fft.fft2(fp)) * np.fft.fft2(gp)
    mag = np.abs(x)
    x = np.where(mag > 0, x / np.where(mag > 0, mag, 1), 0)
    raw = np.fft.fftshift(np.real(np.fft.ifft2(x)))
    half, h = (n - 1) // 2, m // 2
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    return raw[h - (i - half), h + (j - half)]


@pytest.mark.parametrize("n,theta", [(64, 0.0), (64, 0.031), (128, -0.02)])
def test_phase_correlation_restatement_equals_numpy_fft(orc, n, theta):
    rng = np.random.default_rng(n)
    f = rng.random((n, n))
    g = np.roll(f, (3, -4), (0, 1)) + 0.05 * rng.random((n, n))
    cfg = orc.make_config(n_theta=90, delta_theta=np.pi / 90, n_xy=n, delta_xy=0.5, n_radius=0, pad_angle=-1)
    orc.finalize(cfg)
    tx, ty, s = orc.estimate_translation_ex(f, g, theta, cfg, 0.5, 3 * n // 2, True)
    gr = orc.rotate_bilinear(g, -theta)  # rotate_bilinear is pinned to the reference elsewhere
    ref = _phase_corr_numpy(f, gr, n)
    assert np.abs(s - ref).max() <= 1e-12 * np.abs(ref).max()
    if theta == 0.0:  # a pure circular shift: the phase-correlation peak is the shift,
        r, c = np.unravel_index(np.argmax(s), s.shape)  # rows flipped (matcher.cpp:171-182)
        half = (n - 1) // 2
        assert (half - r, c - half) == (3, -4)
