"""C ABI + host logic without a GPU: the library loads, exports every symbol the
headers declare, and the config semantics mirror matcher.cpp:11-37."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fscan_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header", ["fscan_cuda.h", "fscan_synth.h", "fscan_io.h"])
def test_library_exports_every_declared_symbol(fb, header):
    names = declared_functions(header)
    assert len(names) >= 3
    lib = C.CDLL(fb.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header(fb):
    names = set(declared_functions("fscan_cuda.h")) | set(declared_functions("fscan_synth.h")) | \
        set(declared_functions("fscan_io.h"))
    assert names <= set(fb.SYMBOLS), names - set(fb.SYMBOLS)


def test_drop_in_cpp_symbols_exported(fb):
    import subprocess
    out = subprocess.run(["nm", "-DC", fb.LIB_PATH], capture_output=True, text=True).stdout
    for sym in ("fscan::scan_match(fscan::ScanGrid const&, fscan::ScanGrid const&, fscan::MatchConfig const&)",
                "fscan::estimate_rotation(", "fscan::estimate_translation(", "fscan::soft_argmax(",
                "fscan::finalize(fscan::MatchConfig&)", "fscan::validate(fscan::MatchConfig const&)",
                "fscan::scan_match_batch(", "fscan::brute_force_match(", "fscan::timing_comparison(",
                "fscan::kitti_drift(", "fscan::integrate(", "fscan::odometry(", "fscan::read_scan(",
                "fscan::write_scan(", "fscan::read_scans_f32(", "fscan::next_fast_size(int)"):
        assert sym in out, sym


def test_built_for_sm100a(fb):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", fb.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_defaults_finalize_validate(fb):  # test_matcher.cpp:60-103
    cfg = fb.MatchConfig()
    cfg.validate()
    assert (cfg.n_radius, cfg.pad_angle) == (128, 92)
    d = fb.MatchConfig(n_xy=65, n_theta=100, delta_theta=math.pi / 100, n_radius=0, pad_angle=-1).finalize()
    assert (d.n_radius, d.pad_angle) == (33, 13)
    t = fb.MatchConfig(n_theta=2, delta_theta=0.01, pad_angle=-1).finalize()
    assert t.pad_angle == 1
    base = dict(n_xy=65, delta_xy=0.4, n_theta=129, delta_theta=math.pi / 129, n_radius=33, pad_angle=17,
                band_lo=0.15)
    for kw in (dict(band_lo=0.8), dict(delta_theta=math.pi / 64.0), dict(pad_angle=129),
               dict(softargmax_window=0), dict(t_theta=0.0), dict(t_xy=-1.0), dict(n_xy=2),
               dict(delta_xy=0.0), dict(n_radius=1), dict(n_theta=0)):
        with pytest.raises(fb.FscanInvalidArgument):
            fb.MatchConfig(**{**base, **kw}).validate()
    fb.MatchConfig(**{**base, "n_xy": 64}).validate()  # D1: even n accepted


def test_baseline_configs_resolve(fb):
    c1, d1, b1 = fb.baseline_config(1)
    assert (c1.n_xy, c1.n_theta, c1.pad_angle, c1.n_radius, d1, b1) == (256, 360, 45, 128, 0.5, 1)
    c4, d4, b4 = fb.baseline_config(4)
    assert (c4.n_xy, c4.n_theta, c4.pad_angle, c4.n_radius, d4, b4, c4.t_theta) == (512, 720, 90, 256, 0.25, 4096, 1.0)
    c5, d5, b5 = fb.baseline_config(5)
    assert (c5.n_xy, c5.n_theta, c5.pad_angle, c5.n_radius, c5.t_xy) == (1024, 1440, 180, 512, 0.5)


def test_context_without_gpu_fails_loudly(fb):
    """No CPU fallback: on a GPU-less host every compute entry point errors."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("this host has a GPU")
    cfg, _, _ = fb.baseline_config(2)
    with pytest.raises(fb.FscanError) as ei:
        fb.Matcher(cfg, max_batch=1)
    assert ei.value.status in (fb.ERR_NO_DEVICE, fb.ERR_CUDA)


@pytest.mark.parametrize("n", [31, 2048])
def test_unsupported_grid_sizes_are_rejected(fb, n):
    """Grid sides outside [33, 1024] are refused before any device work (odd
    sides such as the reference's default 255 are supported: DESIGN.md §3.9)."""
    cfg = fb.MatchConfig.for_grid(n, 0.4, 733)
    with pytest.raises(fb.FscanError) as ei:
        fb.Matcher(cfg, max_batch=1)
    assert ei.value.status == fb.ERR_UNSUPPORTED


def test_result_struct_layout(fb):
    assert C.sizeof(fb.CPairResult) == 80 == fb.RESULT_DTYPE.itemsize
    assert C.sizeof(fb.CConfig) == 80  # int32/double layout of fscan_config (x86-64 SysV)


def test_shard_ranges_cover_and_partition():
    from paper_2203_00459_b200.shard import shard_range
    for total in (0, 1, 7, 64, 4096, 1023):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0
            assert sum(c for _, c in spans) == total
            for (f0, c0), (f1, _) in zip(spans, spans[1:]):
                assert f0 + c0 == f1
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


# ---- .fscn ingestion (proj/src/io.cpp:84-131, proj/tests/test_io.cpp:33-61); CPU only ----

def test_fscn_round_trip_and_layout(fb, tmp_path):  # test_io.cpp:33-45
    rng = np.random.default_rng(99)
    a = (np.floor(rng.random((17, 17)) * 4096.0) / 256.0).astype(np.float32)  # exact in f32
    path = str(tmp_path / "roundtrip.fscn")
    fb.write_scan(path, a, 0.25)
    assert os.path.getsize(path) == 16 + 17 * 17 * 4
    b, d = fb.read_scans([path])
    assert b.shape == (1, 17, 17) and d[0] == 0.25
    np.testing.assert_array_equal(a, b[0])


def test_fscn_reader_rejects_malformed_files(fb, tmp_path):  # test_io.cpp:47-61
    bad = tmp_path / "bad_magic.fscn"
    bad.write_bytes(b"PNGX0000000000000000")
    with pytest.raises(fb.FscanError, match="bad magic"):
        fb.read_scans([str(bad)])
    tr = str(tmp_path / "truncated.fscn")
    fb.write_scan(tr, np.ones((17, 17), np.float32), 0.25)
    with open(tr, "r+b") as fh:
        fh.truncate(16 + 40)
    with pytest.raises(fb.FscanError, match="truncated"):
        fb.read_scans([tr])
    with pytest.raises(fb.FscanError, match="cannot open"):
        fb.read_scans([str(tmp_path / "does_not_exist.fscn")])


def test_fscn_batch_reads_many_files_in_order(fb, tmp_path):
    grids = [np.full((8, 8), k, np.float32) for k in range(40)]
    paths = []
    for k, g in enumerate(grids):
        paths.append(str(tmp_path / f"s{k:03d}.fscn"))
        fb.write_scan(paths[-1], g, 0.5)
    buf, deltas = fb.read_scans(paths, threads=7)
    assert buf.shape == (40, 8, 8) and (deltas == 0.5).all()
    assert all((buf[k] == k).all() for k in range(40))
    fb.write_scan(str(tmp_path / "odd.fscn"), np.zeros((4, 4), np.float32), 0.5)
    with pytest.raises(fb.FscanError, match="grid size"):
        fb.read_scans(paths + [str(tmp_path / "odd.fscn")])


# ---- .fscn files against the reference's OWN reader / writer (io.cpp:82-131, oracle/_ref) ----

def _ref_or_skip():
    import oracle
    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    return oracle


def test_fscn_reference_writer_to_our_reader_and_back(fb, tmp_path):
    """Files written by the reference's write_scan read bit-identically through
    fscan_fscn_read_batch, and files we write read bit-identically through the
    reference's read_scan (header fields and float32 payload)."""
    orc = _ref_or_skip()
    rng = np.random.default_rng(7)
    grids = [rng.standard_normal((n, n)).astype(np.float32) for n in (33, 64, 64)]
    # reference -> ours
    paths = []
    for k, (g, d) in enumerate(zip(grids[1:], (0.25, 0.125))):
        paths.append(str(tmp_path / f"ref_{k}.fscn"))
        orc.ref_write_scan(paths[-1], g, d)
    buf, deltas = fb.read_scans(paths)
    np.testing.assert_array_equal(buf[0], grids[1])
    np.testing.assert_array_equal(buf[1], grids[2])
    assert list(deltas) == [0.25, 0.125]
    # ours -> reference (odd and even sides; the byte layout is the same)
    for k, (g, d) in enumerate(((grids[0], 0.4), (grids[1], 0.5))):
        p = str(tmp_path / f"ours_{k}.fscn")
        fb.write_scan(p, g, d)
        r, rd = orc.ref_read_scan(p)
        np.testing.assert_array_equal(r, g)
        assert rd == np.float32(d)
        with open(p, "rb") as fh:
            ours = fh.read()
        q = str(tmp_path / f"ref_again_{k}.fscn")
        orc.ref_write_scan(q, g, d)
        with open(q, "rb") as fh:
            assert fh.read() == ours  # byte-identical files


def test_fscn_malformed_files_fail_like_the_reference(fb, tmp_path):
    """Bad magic, truncated payload, implausible size: both readers reject the file
    with the same reason (io.cpp:113-126 messages)."""
    orc = _ref_or_skip()
    bad = tmp_path / "bad.fscn"
    bad.write_bytes(b"PNGX" + b"\0" * 16)
    tr = str(tmp_path / "trunc.fscn")
    orc.ref_write_scan(tr, np.ones((16, 16), np.float32), 0.5)
    with open(tr, "r+b") as fh:
        fh.truncate(16 + 100)
    huge = tmp_path / "huge.fscn"
    huge.write_bytes(b"FSCN" + np.uint32(1 << 16).tobytes() + np.float32(0.5).tobytes() + b"\0" * 4)
    for path, why in ((str(bad), "bad magic"), (tr, "truncated"), (str(huge), "implausible grid size")):
        with pytest.raises(orc.OracleError, match=why):
            orc.ref_read_scan(path)
        with pytest.raises(fb.FscanError, match=why):
            fb.read_scans([path])
