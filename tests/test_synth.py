"""Seeded generator (host side, no GPU): determinism per pair index, pose ranges,
mask range, and that the oracle recovers the generator's ground truth."""
import math

import numpy as np
import pytest

from conftest import oracle_cfg


def test_pairs_are_deterministic_per_index(fb):
    s = fb.synth_spec(2)
    a = fb.synth_pairs_host(s, 0, 3, threads=3)
    b = fb.synth_pairs_host(s, 1, 2, threads=1)  # same pairs 1, 2 from a different batch split
    for x, y in zip(a[:4], b[:4]):
        np.testing.assert_array_equal(x[1:], y)
    np.testing.assert_array_equal(a[4][1:], b[4])


def test_pose_and_mask_ranges(fb):
    for cid in (1, 2, 5):
        s = fb.synth_spec(cid)
        f, g, mf, mg, truth = fb.synth_pairs_host(s, 0, 2)
        assert np.all(np.abs(truth[:, 0]) <= s.theta_max)
        assert np.all(np.abs(truth[:, 1:]) <= s.t_max)
        assert np.all(np.isfinite(f)) and np.all(f >= 0)
        if s.masks:
            assert mf.min() >= 0.0 and mf.max() <= 1.0 and mf.std() > 0.01
        else:
            assert np.all(mf == 1.0)


def test_polar_sweeps_shape_and_conversion(fb):
    s = fb.synth_spec(3)
    pf, pg, truth = fb.synth_polar_host(s, 0, 1)
    assert pf.shape == (1, 400, 3768) and np.all(pf >= 0)
    f, g, mf, mg, t2 = fb.synth_pairs_host(s, 0, 1)
    np.testing.assert_array_equal(truth, t2)
    assert f.shape == (1, 512, 512)


@pytest.mark.parametrize("cid", [2])
def test_oracle_recovers_generator_truth(fb, orc, cid):
    cfg, delta, _ = fb.baseline_config(cid)
    s = fb.synth_spec(cid)
    f, g, mf, mg, truth = fb.synth_pairs_host(s, 0, 3)
    oc = oracle_cfg(orc, cfg)
    for i in range(3):
        r = orc.scan_match(f[i], g[i], oc, delta, mf[i], mg[i])
        assert abs(r.theta - truth[i, 0]) <= 2 * cfg.delta_theta
        assert math.hypot(r.tx - truth[i, 1], r.ty - truth[i, 2]) <= 2 * delta
