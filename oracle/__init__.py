"""CPU parity oracle — TEST INFRASTRUCTURE.

Loads ``oracle/liboracle.so`` (the C restatement, ``fo_*``) and, when it has
been built, ``oracle/_ref/libfscan_ref.so`` (the reference's own sources,
``ref_*``). Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline legs import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_ORACLE = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libfscan_ref.so")
LIB_GEN = os.path.join(HERE, "libsynth_gen.so")
REF_SRC = "/root/reference/proj"


class FoConfig(C.Structure):
    _fields_ = [
        ("n_theta", C.c_int), ("delta_theta", C.c_double), ("t_theta", C.c_double),
        ("n_xy", C.c_int), ("delta_xy", C.c_double), ("t_xy", C.c_double),
        ("band_lo", C.c_double), ("band_hi", C.c_double),
        ("n_radius", C.c_int), ("pad_angle", C.c_int),
        ("softargmax_window", C.c_int), ("normalize_scores", C.c_int),
    ]


class FoResult(C.Structure):
    _fields_ = [
        ("theta", C.c_double), ("tx", C.c_double), ("ty", C.c_double),
        ("theta_hard", C.c_double), ("theta_peak", C.c_double),
        ("xy_hard_x", C.c_double), ("xy_hard_y", C.c_double), ("xy_peak", C.c_double),
        ("theta_bin", C.c_int), ("xy_row", C.c_int), ("xy_col", C.c_int), ("pad_", C.c_int),
    ]


class FoBfResult(C.Structure):
    _fields_ = [
        ("theta", C.c_double), ("tx", C.c_double), ("ty", C.c_double), ("score", C.c_double),
        ("theta_index", C.c_int), ("xy_row", C.c_int), ("xy_col", C.c_int), ("pad_", C.c_int),
    ]


def build(ref: bool = True) -> None:
    """Build liboracle.so (and _ref when the reference tree is present)."""
    target = "all" if (ref and os.path.isdir(REF_SRC)) else "oracle"
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


_libs: dict[str, C.CDLL] = {}

_D = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_F = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")


def _declare(lib: C.CDLL, prefix: str) -> None:
    dp = C.POINTER(C.c_double)
    for name, args in {
        "band_magnitude": [dp, C.c_int, C.c_double, C.c_double, dp],
        "cart2pol": [dp, C.c_int, C.c_int, C.c_int, C.c_double, dp],
        "rotate_bilinear": [dp, C.c_int, C.c_double, dp],
        "xcorr": [dp, dp, C.c_int, C.c_int, dp],
        "soft_argmax": [dp, C.c_int, C.c_int, dp, dp, C.c_double, C.c_int, C.c_int, dp, dp],
        "scan_match": [dp, dp, dp, dp, C.c_int, C.c_double, C.POINTER(FoConfig),
                       C.POINTER(FoResult), dp, dp, C.c_char_p, C.c_int],
    }.items():
        fn = getattr(lib, f"{prefix}_{name}")
        fn.argtypes = args
        fn.restype = C.c_int


def lib(which: str = "oracle") -> C.CDLL:
    """which = 'oracle' (restatement) or 'ref' (the reference's own code)."""
    if which in _libs:
        return _libs[which]
    path = LIB_ORACLE if which == "oracle" else LIB_REF
    if not os.path.exists(path):
        build(ref=(which == "ref"))
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} is not built (reference tree absent?)")
    L = C.CDLL(path)
    prefix = "fo" if which == "oracle" else "ref"
    _declare(L, prefix)
    if which == "oracle":
        L.fo_finalize.argtypes = [C.POINTER(FoConfig)]
        L.fo_finalize.restype = None
        L.fo_validate.argtypes = [C.POINTER(FoConfig), C.c_char_p, C.c_int]
        L.fo_validate.restype = C.c_int
        L.fo_next_fast_size.argtypes = [C.c_int]
        L.fo_next_fast_size.restype = C.c_int
        L.fo_polar_to_cart.argtypes = [C.POINTER(C.c_double), C.c_int, C.c_int, C.c_double,
                                       C.c_int, C.c_double, C.POINTER(C.c_double)]
        L.fo_polar_to_cart.restype = C.c_int
        L.fo_brute_force.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int, C.c_double,
                                     C.POINTER(C.c_double), C.c_int, C.POINTER(FoBfResult)]
        L.fo_brute_force.restype = C.c_int
        L.fo_estimate_translation_ex.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int, C.c_double,
                                                 C.c_double, C.POINTER(FoConfig), C.c_int, C.c_int,
                                                 C.POINTER(C.c_double), C.POINTER(C.c_double),
                                                 C.POINTER(C.c_double)]
        L.fo_estimate_translation_ex.restype = C.c_int
    else:
        L.ref_brute_force.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int, C.c_double,
                                      C.POINTER(C.c_double), C.c_int, C.POINTER(FoBfResult), C.c_char_p,
                                      C.c_int]
        L.ref_brute_force.restype = C.c_int
        L.ref_verify.argtypes = [C.c_char_p, C.c_int]
        L.ref_verify.restype = C.c_int
        L.ref_scan_match_batch_f32.argtypes = [
            C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(C.c_float),
            C.c_int, C.c_int, C.c_double, C.POINTER(FoConfig), C.c_int, C.POINTER(FoResult)]
        L.ref_scan_match_batch_f32.restype = C.c_int
        L.ref_write_scan.argtypes = [C.c_char_p, C.POINTER(C.c_float), C.c_int, C.c_double, C.c_char_p, C.c_int]
        L.ref_write_scan.restype = C.c_int
        L.ref_read_scan.argtypes = [C.c_char_p, C.POINTER(C.c_float), C.c_int, C.POINTER(C.c_int),
                                    C.POINTER(C.c_double), C.c_char_p, C.c_int]
        L.ref_read_scan.restype = C.c_int
    _libs[which] = L
    return L


def have_ref() -> bool:
    try:
        lib("ref")
        return True
    except (FileNotFoundError, OSError, subprocess.CalledProcessError):
        return False


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _pf(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_float))


def make_config(**kw) -> FoConfig:
    """MatchConfig with the reference defaults (matcher.hpp:13-26), overridden by kw."""
    d = dict(n_theta=733, delta_theta=np.pi / 733.0, t_theta=2.0, n_xy=255, delta_xy=0.4,
             t_xy=1.0, band_lo=0.03, band_hi=0.75, n_radius=128, pad_angle=92,
             softargmax_window=16, normalize_scores=1)
    d.update(kw)
    d["normalize_scores"] = int(bool(d["normalize_scores"]))
    return FoConfig(**d)


def finalize(cfg: FoConfig) -> FoConfig:
    lib("oracle").fo_finalize(C.byref(cfg))
    return cfg


@dataclass
class MatchOut:
    theta: float
    tx: float
    ty: float
    theta_hard: float
    theta_peak: float
    xy_hard: tuple
    xy_peak: float
    theta_bin: int
    xy_row: int
    xy_col: int
    theta_surface: np.ndarray
    xy_surface: np.ndarray


class OracleError(ValueError):
    pass


def scan_match(f, g, cfg: FoConfig, delta: float, mf=None, mg=None, which: str = "oracle") -> MatchOut:
    """Run the oracle's scan_match on float64 copies of the inputs."""
    L = lib(which)
    n = int(f.shape[0])
    f = np.ascontiguousarray(f, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    mf = None if mf is None else np.ascontiguousarray(mf, dtype=np.float64)
    mg = None if mg is None else np.ascontiguousarray(mg, dtype=np.float64)
    ts = np.zeros(max(cfg.n_theta, 1), dtype=np.float64)
    xs = np.zeros((n, n), dtype=np.float64)
    res = FoResult()
    err = C.create_string_buffer(512)
    fn = L.fo_scan_match if which == "oracle" else L.ref_scan_match
    rc = fn(_p(f), _p(g), _p(mf), _p(mg), n, delta, C.byref(cfg), C.byref(res), _p(ts), _p(xs), err, 512)
    if rc != 0:
        raise OracleError(err.value.decode())
    return MatchOut(res.theta, res.tx, res.ty, res.theta_hard, res.theta_peak,
                    (res.xy_hard_x, res.xy_hard_y), res.xy_peak, res.theta_bin,
                    res.xy_row, res.xy_col, ts, xs)


def brute_force(f, g, thetas, delta: float, which: str = "oracle") -> FoBfResult:
    """brute_force_match (oracle.cpp:40-67) on float64 copies of the inputs."""
    L = lib(which)
    n = int(f.shape[0])
    f = np.ascontiguousarray(f, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    th = np.ascontiguousarray(thetas, dtype=np.float64)
    res = FoBfResult()
    if which == "oracle":
        rc = L.fo_brute_force(_p(f), _p(g), n, delta, _p(th), int(th.size), C.byref(res))
        if rc != 0:
            raise OracleError("brute_force_match: empty theta candidate list")
    else:
        err = C.create_string_buffer(512)
        rc = L.ref_brute_force(_p(f), _p(g), n, delta, _p(th), int(th.size), C.byref(res), err, 512)
        if rc != 0:
            raise OracleError(err.value.decode())
    return res


def estimate_translation_ex(f, g, theta, cfg: FoConfig, delta: float, pad_size: int = 0, phase: bool = False):
    """Translation stage with padded size pad_size (0: the reference's) and optional
    phase correlation (restatement only): (tx, ty, surface)."""
    L = lib("oracle")
    n = int(f.shape[0])
    f = np.ascontiguousarray(f, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    s = np.zeros((n, n))
    tx, ty = C.c_double(), C.c_double()
    L.fo_estimate_translation_ex(_p(f), _p(g), n, delta, float(theta), C.byref(cfg), int(pad_size), int(phase),
                                 C.byref(tx), C.byref(ty), _p(s))
    return tx.value, ty.value, s


def band_magnitude(img, band_lo, band_hi, which="oracle"):
    img = np.ascontiguousarray(img, dtype=np.float64)
    out = np.zeros_like(img)
    fn = getattr(lib(which), f"{'fo' if which == 'oracle' else 'ref'}_band_magnitude")
    assert fn(_p(img), img.shape[0], band_lo, band_hi, _p(out)) == 0
    return out


def cart2pol(a, n_angle, n_radius, span, which="oracle"):
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = np.zeros((n_angle, n_radius))
    fn = getattr(lib(which), f"{'fo' if which == 'oracle' else 'ref'}_cart2pol")
    assert fn(_p(a), a.shape[0], n_angle, n_radius, span, _p(out)) == 0
    return out


def rotate_bilinear(g, theta, which="oracle"):
    g = np.ascontiguousarray(g, dtype=np.float64)
    out = np.zeros_like(g)
    fn = getattr(lib(which), f"{'fo' if which == 'oracle' else 'ref'}_rotate_bilinear")
    assert fn(_p(g), g.shape[0], theta, _p(out)) == 0
    return out


def xcorr(a, b, which="oracle"):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = np.zeros_like(a)
    fn = getattr(lib(which), f"{'fo' if which == 'oracle' else 'ref'}_xcorr")
    assert fn(_p(a), _p(b), a.shape[0], a.shape[1], _p(out)) == 0
    return out


def soft_argmax(scores, row_coords, col_coords, gain, window, normalize=True, which="oracle"):
    s = np.ascontiguousarray(scores, dtype=np.float64)
    rc = np.ascontiguousarray(row_coords, dtype=np.float64)
    cc = np.ascontiguousarray(col_coords, dtype=np.float64)
    r, c = C.c_double(), C.c_double()
    fn = getattr(lib(which), f"{'fo' if which == 'oracle' else 'ref'}_soft_argmax")
    assert fn(_p(s), s.shape[0], s.shape[1], _p(rc), _p(cc), gain, window, int(normalize),
              C.byref(r), C.byref(c)) == 0
    return r.value, c.value


def polar_to_cart(polar, range_res, n, delta):
    p = np.ascontiguousarray(polar, dtype=np.float64)
    out = np.zeros((n, n))
    assert lib("oracle").fo_polar_to_cart(_p(p), p.shape[0], p.shape[1], range_res, n, delta, _p(out)) == 0
    return out


def ref_verify() -> tuple[int, str]:
    buf = C.create_string_buffer(8192)
    fails = lib("ref").ref_verify(buf, 8192)
    return fails, buf.value.decode()


def ref_batch_f32(f, g, mf, mg, cfg: FoConfig, delta: float, threads: int):
    """Reference scan_match over a batch with parallel_for (CPU baseline)."""
    f = np.ascontiguousarray(f, dtype=np.float32)
    g = np.ascontiguousarray(g, dtype=np.float32)
    mf = None if mf is None else np.ascontiguousarray(mf, dtype=np.float32)
    mg = None if mg is None else np.ascontiguousarray(mg, dtype=np.float32)
    b, n = f.shape[0], f.shape[1]
    out = (FoResult * b)()
    rc = lib("ref").ref_scan_match_batch_f32(_pf(f), _pf(g), _pf(mf), _pf(mg), b, n, delta,
                                             C.byref(cfg), threads, out)
    if rc != 0:
        raise OracleError(f"ref batch failed rc={rc}")
    return out


# ---------------------------------------------------------------- inputs for the CPU arm
# bench.py's reference arm must not map the product library; it builds its
# inputs with libsynth_gen.so (the product's host renderer compiled on its own,
# oracle/Makefile) and its configs with the restated finalize (fo_finalize).

class SynthSpec(C.Structure):
    """fscan_synth_spec (include/fscan_synth.h)."""
    _fields_ = [
        ("polar", C.c_int), ("n", C.c_int), ("delta", C.c_double),
        ("n_reflectors", C.c_int), ("n_segments", C.c_int),
        ("sigma_lo_px", C.c_double), ("sigma_hi_px", C.c_double), ("seg_sigma_px", C.c_double),
        ("extent_frac", C.c_double), ("theta_max", C.c_double), ("t_max", C.c_double),
        ("speckle", C.c_double), ("masks", C.c_int), ("mask_sigma", C.c_double),
        ("n_az", C.c_int), ("n_range", C.c_int), ("range_res", C.c_double), ("att_r0", C.c_double),
        ("seed", C.c_uint64),
    ]


def gen_lib() -> C.CDLL:
    if "gen" in _libs:
        return _libs["gen"]
    if not os.path.exists(LIB_GEN):
        build(ref=False)
    L = C.CDLL(LIB_GEN)
    L.fscan_synth_preset.argtypes = [C.c_int, C.POINTER(SynthSpec)]
    L.fscan_synth_preset.restype = C.c_int
    L.fscan_synth_pairs_host.argtypes = [C.POINTER(SynthSpec), C.c_int, C.c_int] + [C.c_void_p] * 5 + [C.c_int]
    L.fscan_synth_pairs_host.restype = C.c_int
    _libs["gen"] = L
    return L


def synth_pairs_host(config_id: int, first: int, count: int, threads: int = 0, **overrides):
    """(f, g, mf, mg, truth) of BASELINE config `config_id`, pairs [first, first + count)."""
    L = gen_lib()
    spec = SynthSpec()
    if L.fscan_synth_preset(int(config_id), C.byref(spec)) != 0:
        raise ValueError(f"unknown config {config_id}")
    for k, v in overrides.items():
        setattr(spec, k, v)
    n = spec.n
    f = np.empty((count, n, n), np.float32)
    g, mf, mg = np.empty_like(f), np.empty_like(f), np.empty_like(f)
    truth = np.empty((count, 3), np.float64)
    rc = L.fscan_synth_pairs_host(C.byref(spec), first, count, f.ctypes.data, g.ctypes.data, mf.ctypes.data,
                                  mg.ctypes.data, truth.ctypes.data, int(threads))
    if rc:
        raise RuntimeError(f"fscan_synth_pairs_host failed ({rc})")
    return f, g, mf, mg, truth


# (n, grid delta [m], n_theta, t_theta = t_xy or None for the defaults, batch) of
# BASELINE.json configs 1..5
BASELINE = {1: (256, 0.5, 360, None, 1), 2: (256, 0.5, 360, 1.0, 64), 3: (512, 0.25, 720, 1.0, 64),
            4: (512, 0.25, 720, 1.0, 4096), 5: (1024, 0.125, 1440, 0.5, 1024)}


def baseline_config(cid: int) -> tuple[FoConfig, float, int]:
    """(finalized FoConfig, grid delta, batch) of BASELINE config `cid` (delta_theta =
    pi / n_theta, n_radius / pad_angle resolved by finalize, matcher.cpp:11-15)."""
    n, delta, nt, t, batch = BASELINE[cid]
    kw = dict(n_theta=nt, delta_theta=np.pi / nt, n_xy=n, delta_xy=delta, n_radius=0, pad_angle=-1)
    if t is not None:
        kw.update(t_theta=t, t_xy=t)
    return finalize(make_config(**kw)), delta, batch


def host_descriptor() -> dict:
    """CPU model + logical core count (the reference's host_descriptor, bench.cpp:84-105)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "logical_cores": os.cpu_count() or 1}


def ref_write_scan(path: str, grid, delta: float) -> None:
    """The reference's own write_scan (io.cpp:82-100)."""
    g = np.ascontiguousarray(grid, dtype=np.float32)
    err = C.create_string_buffer(512)
    if lib("ref").ref_write_scan(os.fsencode(path), _pf(g), int(g.shape[0]), float(delta), err, 512) != 0:
        raise OracleError(err.value.decode())


def ref_read_scan(path: str, n_max: int = 4096):
    """The reference's own read_scan (io.cpp:102-131): (float32 grid, delta)."""
    buf = np.empty(n_max * n_max, np.float32)
    n, d = C.c_int(), C.c_double()
    err = C.create_string_buffer(512)
    if lib("ref").ref_read_scan(os.fsencode(path), _pf(buf), n_max, C.byref(n), C.byref(d), err, 512) != 0:
        raise OracleError(err.value.decode())
    return buf[: n.value * n.value].reshape(n.value, n.value).copy(), d.value
