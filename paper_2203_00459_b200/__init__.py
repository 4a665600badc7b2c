"""B200-native decoupled Fourier pose search (f-MbyM, arXiv 2203.00459).

Python host side of the drop-in for the reference hot path
``fscan::scan_match`` (proj/src/matcher.cpp:189-216) and its pybind11 binding
``fscan.scan_match(f, g, delta, config)`` (proj/python/module.cpp:117-136).
Everything computes in the sm_100a kernels of ``libfscan_b200.so`` through the
C ABI declared in ``include/fscan_cuda.h``; this module only marshals
pointers. There is no CPU fallback: without the library or a B200 every
compute call raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
# FSCAN_LIB: load an alternative build of the same library for A/B kernel timing;
# only builds under <repo>/ab/ (tools/ab_build.sh) are accepted, and bench.py
# records the path it loaded
_AB_DIR = os.path.join(ROOT, "ab") + os.sep
_ENV_LIB = os.environ.get("FSCAN_LIB")
if _ENV_LIB and not os.path.abspath(_ENV_LIB).startswith(_AB_DIR):
    raise RuntimeError(f"FSCAN_LIB must point at an A/B build under {_AB_DIR} (got {_ENV_LIB})")
LIB_PATH = os.path.abspath(_ENV_LIB) if _ENV_LIB else os.path.join(HERE, "libfscan_b200.so")

OK, ERR_INVALID_ARGUMENT, ERR_NONFINITE, ERR_MASK_RANGE, ERR_UNSUPPORTED, ERR_CUDA, ERR_NO_DEVICE, ERR_IO = range(8)
_STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "NONFINITE", 3: "MASK_RANGE", 4: "UNSUPPORTED",
           5: "CUDA", 6: "NO_DEVICE", 7: "IO"}


class FscanError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{_STATUS.get(status, status)}] {msg}")
        self.status = status


class FscanInvalidArgument(FscanError, ValueError):
    """std::invalid_argument of the reference (bad config, NaN/Inf, mask range)."""


def _raise(status: int, msg: str):
    if status in (ERR_INVALID_ARGUMENT, ERR_NONFINITE, ERR_MASK_RANGE):
        raise FscanInvalidArgument(status, msg)
    raise FscanError(status, msg)


class CConfig(C.Structure):
    _fields_ = [
        ("n_theta", C.c_int32), ("delta_theta", C.c_double), ("t_theta", C.c_double),
        ("n_xy", C.c_int32), ("delta_xy", C.c_double), ("t_xy", C.c_double),
        ("band_lo", C.c_double), ("band_hi", C.c_double),
        ("n_radius", C.c_int32), ("pad_angle", C.c_int32),
        ("softargmax_window", C.c_int32), ("normalize_scores", C.c_int32),
    ]


class CPairResult(C.Structure):
    _fields_ = [
        ("theta", C.c_double), ("tx", C.c_double), ("ty", C.c_double),
        ("theta_hard", C.c_double), ("theta_peak", C.c_double),
        ("xy_hard_x", C.c_double), ("xy_hard_y", C.c_double), ("xy_peak", C.c_double),
        ("theta_bin", C.c_int32), ("xy_row", C.c_int32), ("xy_col", C.c_int32), ("status", C.c_int32),
    ]


RESULT_DTYPE = np.dtype([
    ("theta", "f8"), ("tx", "f8"), ("ty", "f8"), ("theta_hard", "f8"), ("theta_peak", "f8"),
    ("xy_hard_x", "f8"), ("xy_hard_y", "f8"), ("xy_peak", "f8"),
    ("theta_bin", "i4"), ("xy_row", "i4"), ("xy_col", "i4"), ("status", "i4")])
assert RESULT_DTYPE.itemsize == C.sizeof(CPairResult)


class CBfResult(C.Structure):
    _fields_ = [
        ("theta", C.c_double), ("tx", C.c_double), ("ty", C.c_double), ("score", C.c_double),
        ("theta_index", C.c_int32), ("xy_row", C.c_int32), ("xy_col", C.c_int32), ("status", C.c_int32),
    ]


BF_DTYPE = np.dtype([("theta", "f8"), ("tx", "f8"), ("ty", "f8"), ("score", "f8"),
                     ("theta_index", "i4"), ("xy_row", "i4"), ("xy_col", "i4"), ("status", "i4")])
assert BF_DTYPE.itemsize == C.sizeof(CBfResult)


class CSynthSpec(C.Structure):
    _fields_ = [
        ("polar", C.c_int), ("n", C.c_int), ("delta", C.c_double),
        ("n_reflectors", C.c_int), ("n_segments", C.c_int),
        ("sigma_lo_px", C.c_double), ("sigma_hi_px", C.c_double), ("seg_sigma_px", C.c_double),
        ("extent_frac", C.c_double), ("theta_max", C.c_double), ("t_max", C.c_double),
        ("speckle", C.c_double), ("masks", C.c_int), ("mask_sigma", C.c_double),
        ("n_az", C.c_int), ("n_range", C.c_int), ("range_res", C.c_double), ("att_r0", C.c_double),
        ("seed", C.c_uint64),
    ]


def build(force: bool = False) -> str:
    """Compile libfscan_b200.so for sm_100a (nvcc cross-compiles without a GPU)."""
    cmd = ["make", "-s", "-C", os.path.join(HERE, "csrc")]
    if force:
        subprocess.run(cmd + ["clean"], check=True)
    subprocess.run(cmd + ["-j8"], check=True)
    return LIB_PATH


_lib: C.CDLL | None = None

_P = C.c_void_p
SYMBOLS = {
    # name: (restype, argtypes)
    "fscan_config_defaults": (None, [C.POINTER(CConfig)]),
    "fscan_config_finalize": (None, [C.POINTER(CConfig)]),
    "fscan_config_validate": (C.c_int, [C.POINTER(CConfig), C.c_char_p, C.c_size_t]),
    "fscan_ctx_create": (C.c_int, [C.c_int, C.POINTER(CConfig), C.c_int, C.POINTER(_P)]),
    "fscan_ctx_destroy": (None, [_P]),
    "fscan_ctx_last_error": (C.c_char_p, [_P]),
    "fscan_ctx_n": (C.c_int, [_P]),
    "fscan_ctx_set_chunk": (C.c_int, [_P, C.c_int]),
    "fscan_match_batch": (C.c_int, [_P, _P, _P, _P, _P, C.c_int, C.c_double, _P, _P, _P, _P]),
    "fscan_match_batch_host": (C.c_int, [_P, _P, _P, _P, _P, C.c_int, C.c_double, _P, _P, _P]),
    "fscan_match_batch_polar": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_double, _P, _P, C.c_int, C.c_double,
                                          _P, _P, _P, _P]),
    "fscan_estimate_rotation_batch": (C.c_int, [_P, _P, _P, C.c_int, _P, _P, _P]),
    "fscan_estimate_translation_batch": (C.c_int, [_P, _P, _P, C.c_int, C.c_double, _P, _P, _P, _P]),
    "fscan_band_magnitude_batch": (C.c_int, [_P, _P, C.c_int, _P, _P]),
    "fscan_brute_force_batch": (C.c_int, [_P, _P, _P, C.c_int, _P, C.c_int, C.c_double, _P, _P]),
    "fscan_odometry_batch": (C.c_int, [_P, _P, _P, C.c_int, C.c_double, _P, _P, _P, _P]),
    "fscan_polar_to_cart_batch": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                            C.c_double, _P, _P]),
    "fscan_check_results": (C.c_int, [_P, C.c_int, _P, C.POINTER(C.c_int)]),
    "fscan_ctx_launches_last": (C.c_int, [_P]),
    "fscan_ctx_rot_columns": (C.c_int, [_P]),
    "fscan_ctx_set_profiling": (C.c_int, [_P, C.c_int]),
    "fscan_ctx_set_graphs": (C.c_int, [_P, C.c_int]),
    "fscan_ctx_graph_stats": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "fscan_ctx_set_phase_correlation": (C.c_int, [_P, C.c_int]),
    "fscan_ctx_kernel_times": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_int]),
    "fscan_fscn_read_header": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_double), C.c_char_p,
                                         C.c_size_t]),
    "fscan_fscn_read_batch": (C.c_int, [C.POINTER(C.c_char_p), C.c_int, C.c_int, _P, _P, C.c_int, C.c_char_p,
                                        C.c_size_t]),
    "fscan_fscn_write": (C.c_int, [C.c_char_p, _P, C.c_int, C.c_double, C.c_char_p, C.c_size_t]),
    "fscan_synth_preset": (C.c_int, [C.c_int, C.POINTER(CSynthSpec)]),
    "fscan_synth_pairs_host": (C.c_int, [C.POINTER(CSynthSpec), C.c_int, C.c_int, _P, _P, _P, _P, _P,
                                         C.c_int]),
    "fscan_synth_polar_host": (C.c_int, [C.POINTER(CSynthSpec), C.c_int, C.c_int, _P, _P, _P, C.c_int]),
    "fscan_synth_pairs_device": (C.c_int, [C.POINTER(CSynthSpec), C.c_int, C.c_int, _P, _P, _P, _P, _P,
                                           _P]),
    "fscan_synth_polar_device": (C.c_int, [C.POINTER(CSynthSpec), C.c_int, C.c_int, _P, _P, _P, _P]),
    "fscan_synth_sequence_device": (C.c_int, [C.POINTER(CSynthSpec), C.c_int, C.c_int, _P, _P, _P, _P]),
}


def lib() -> C.CDLL:
    """Load (building if needed) the native library. Raises if it cannot."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        build()
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in SYMBOLS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


# ---------------------------------------------------------------- config

@dataclass
class MatchConfig:
    """fscan::MatchConfig (matcher.hpp:13-26) with the reference defaults."""
    n_theta: int = 733
    delta_theta: float = math.pi / 733.0
    t_theta: float = 2.0
    n_xy: int = 255
    delta_xy: float = 0.4
    t_xy: float = 1.0
    band_lo: float = 0.03
    band_hi: float = 0.75
    n_radius: int = 128
    pad_angle: int = 92
    softargmax_window: int = 16
    normalize_scores: bool = True

    def to_c(self) -> CConfig:
        return CConfig(int(self.n_theta), float(self.delta_theta), float(self.t_theta), int(self.n_xy),
                       float(self.delta_xy), float(self.t_xy), float(self.band_lo), float(self.band_hi),
                       int(self.n_radius), int(self.pad_angle), int(self.softargmax_window),
                       int(bool(self.normalize_scores)))

    def finalize(self) -> "MatchConfig":
        """matcher.cpp:11-15, in place; returns self."""
        c = self.to_c()
        lib().fscan_config_finalize(C.byref(c))
        self.n_radius, self.pad_angle = c.n_radius, c.pad_angle
        return self

    def validate(self) -> None:
        """matcher.cpp:17-37 (odd-n rule excepted)."""
        c = self.to_c()
        buf = C.create_string_buffer(256)
        st = lib().fscan_config_validate(C.byref(c), buf, 256)
        if st:
            _raise(st, buf.value.decode())

    @staticmethod
    def for_grid(n: int, delta: float, n_theta: int, **kw) -> "MatchConfig":
        """BASELINE-style config: delta_theta = pi/n_theta, sentinels resolved."""
        cfg = MatchConfig(n_theta=n_theta, delta_theta=math.pi / n_theta, n_xy=n, delta_xy=delta,
                          n_radius=0, pad_angle=-1, **kw)
        return cfg.finalize()


# BASELINE.json configs 1..5
def baseline_config(cid: int) -> tuple[MatchConfig, float, int]:
    """(config, grid delta in metres, batch) for BASELINE config 1..5."""
    if cid in (1, 2):
        t = 1.0 if cid == 2 else None
        cfg = MatchConfig.for_grid(256, 0.5, 360)
        if t is not None:
            cfg.t_theta = cfg.t_xy = t
        return cfg, 0.5, (1 if cid == 1 else 64)
    if cid in (3, 4):
        cfg = MatchConfig.for_grid(512, 0.25, 720, t_theta=1.0, t_xy=1.0)
        return cfg, 0.25, (64 if cid == 3 else 4096)
    if cid == 5:
        cfg = MatchConfig.for_grid(1024, 0.125, 1440, t_theta=0.5, t_xy=0.5)
        return cfg, 0.125, 1024
    raise ValueError(cid)


# ---------------------------------------------------------------- matcher

def _ptr(t) -> int | None:
    """Device pointer of a CUDA torch tensor, or of any CUDA array exporting
    __dlpack__ (CuPy, JAX, ...: viewed zero-copy through torch.from_dlpack)."""
    if t is None:
        return None
    if not hasattr(t, "is_cuda") and hasattr(t, "__dlpack__"):
        import torch
        t = torch.from_dlpack(t)
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


def _as_tensor(x):
    """torch view of a foreign CUDA array exporting __dlpack__ (zero-copy); other
    inputs pass through."""
    if x is not None and not hasattr(x, "is_cuda") and hasattr(x, "__dlpack__"):
        import torch
        return torch.from_dlpack(x)
    return x


def _check_tensor(t, name: str, shape: tuple, dtype: str = "float32"):
    """Reject a CUDA input/output the kernels would read or write out of bounds:
    wrong dtype, wrong shape, or (outputs given as raw bytes) too few bytes."""
    if t is None:
        return
    if str(t.dtype).replace("torch.", "") != dtype:
        raise ValueError(f"{name}: expected dtype {dtype}, got {t.dtype}")
    if tuple(int(x) for x in t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")


def _check_bytes(t, name: str, nbytes: int):
    """An output buffer must hold at least nbytes (any dtype, contiguous)."""
    if t is None:
        return
    have = t.numel() * t.element_size()
    if have < nbytes:
        raise ValueError(f"{name}: buffer holds {have} bytes, needs {nbytes}")


def _stream_ptr(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


class Matcher:
    """One device context: a finalized config, tables, workspace and streams."""

    def __init__(self, cfg: MatchConfig, max_batch: int, device: int = 0, chunk: int = 0):
        self.cfg = cfg
        self.device = device
        self.max_batch = max_batch
        h = C.c_void_p()
        c = cfg.to_c()
        st = lib().fscan_ctx_create(device, C.byref(c), max_batch, C.byref(h))
        self._h = h
        if st != OK:
            msg = lib().fscan_ctx_last_error(h).decode() if h.value else ""
            self.close()
            _raise(st, f"fscan_ctx_create: {msg}")
        self.n = lib().fscan_ctx_n(h)
        if chunk:
            self.set_chunk(chunk)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().fscan_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int, what: str):
        if st != OK:
            _raise(st, f"{what}: {lib().fscan_ctx_last_error(self._h).decode()}")

    def set_chunk(self, pairs: int):
        self._check(lib().fscan_ctx_set_chunk(self._h, int(pairs)), "set_chunk")

    @property
    def launches_last(self) -> int:
        return lib().fscan_ctx_launches_last(self._h)

    @property
    def rot_columns(self) -> int:
        """Spectrum columns u < W the rotation stage keeps (fscan_ctx_rot_columns)."""
        return lib().fscan_ctx_rot_columns(self._h)

    KERNELS = ("rot_rows", "rot_cols", "rot_polar", "theta_in", "xlat_rows", "xlat_cols", "xlat_out",
               "finalize", "rot_gather", "polar_to_cart", "mag_unpack", "bf_items", "bf_final",
               "xlat_win")

    def set_phase_correlation(self, on: bool):
        """Opt-in phase correlation in the translation stage (fscan_cuda.h)."""
        self._check(lib().fscan_ctx_set_phase_correlation(self._h, int(bool(on))), "set_phase_correlation")

    def set_graphs(self, on: bool):
        """CUDA-graph replay of repeated identical calls (fscan_ctx_set_graphs)."""
        self._check(lib().fscan_ctx_set_graphs(self._h, int(bool(on))), "set_graphs")

    def graph_stats(self) -> tuple:
        """(captures, replays) of the graph cache."""
        c, r = C.c_int(), C.c_int()
        self._check(lib().fscan_ctx_graph_stats(self._h, C.byref(c), C.byref(r)), "graph_stats")
        return c.value, r.value

    def set_profiling(self, on: bool):
        self._check(lib().fscan_ctx_set_profiling(self._h, int(bool(on))), "set_profiling")

    def kernel_times(self) -> dict:
        """{kernel: (total_ms, launches)} of the last call made in profiling mode."""
        k = len(self.KERNELS)
        ms = (C.c_double * k)()
        cnt = (C.c_int * k)()
        self._check(lib().fscan_ctx_kernel_times(self._h, ms, cnt, k), "kernel_times")
        return {name: (ms[i], cnt[i]) for i, name in enumerate(self.KERNELS) if cnt[i]}

    def match_device(self, f, g, mf=None, mg=None, *, delta: float, out=None, theta_surface=None,
                     xy_surface=None, stream=None):
        """Asynchronous batched scan_match on CUDA tensors [B, N, N] float32.

        ``out`` is a uint8 CUDA tensor of B * sizeof(result) bytes (allocated if
        None) and is returned; decode with :func:`decode_results` after sync.
        """
        f, g, mf, mg = _as_tensor(f), _as_tensor(g), _as_tensor(mf), _as_tensor(mg)
        import torch
        b = int(f.shape[0])
        self._check_pairs(b, f=f, g=g, mf=mf, mg=mg)
        if out is None:
            out = torch.empty(b * RESULT_DTYPE.itemsize, dtype=torch.uint8, device=f.device)
        self._check_outputs(b, out, theta_surface, xy_surface)
        st = lib().fscan_match_batch(self._h, _ptr(f), _ptr(g), _ptr(mf), _ptr(mg), b, float(delta),
                                     _ptr(out), _ptr(theta_surface), _ptr(xy_surface), _stream_ptr(stream))
        self._check(st, "fscan_match_batch")
        return out

    def _check_pairs(self, b: int, **grids):
        """Every grid [b, n, n] float32 (masks both or neither; the reference
        throws 'grid specs differ' for mismatched grids)."""
        if b > self.max_batch:
            raise ValueError(f"batch {b} exceeds the context's max_batch {self.max_batch}")
        if ("mf" in grids) and ((grids["mf"] is None) != (grids.get("mg") is None)):
            raise ValueError("masks: pass both mf and mg, or neither")
        for name, t in grids.items():
            _check_tensor(t, name, (b, self.n, self.n))

    def _check_outputs(self, b: int, out, theta_surface=None, xy_surface=None):
        _check_bytes(out, "out", b * RESULT_DTYPE.itemsize)
        if theta_surface is not None:
            if str(theta_surface.dtype) != "torch.float64":
                raise ValueError(f"theta_surface: expected dtype float64, got {theta_surface.dtype}")
            _check_bytes(theta_surface, "theta_surface", b * max(1, self.cfg.n_theta) * 8)
        if xy_surface is not None:
            _check_tensor(xy_surface, "xy_surface", (b, self.n, self.n))

    def match_polar(self, pf, pg, mf=None, mg=None, *, range_res: float, delta: float, out=None,
                    theta_surface=None, xy_surface=None, stream=None):
        """Config-3 path: raw polar sweeps [B, n_az, n_range] (CUDA tensors) -> K0 -> match."""
        pf, pg, mf, mg = _as_tensor(pf), _as_tensor(pg), _as_tensor(mf), _as_tensor(mg)
        import torch
        if pf.dim() != 3:
            raise ValueError("pf: expected [B, n_az, n_range]")
        b, n_az, n_range = (int(x) for x in pf.shape)
        _check_tensor(pf, "pf", (b, n_az, n_range))
        _check_tensor(pg, "pg", (b, n_az, n_range))
        self._check_pairs(b, mf=mf, mg=mg)
        if out is None:
            out = torch.empty(b * RESULT_DTYPE.itemsize, dtype=torch.uint8, device=pf.device)
        self._check_outputs(b, out, theta_surface, xy_surface)
        st = lib().fscan_match_batch_polar(self._h, _ptr(pf), _ptr(pg), n_az, n_range, float(range_res), _ptr(mf),
                                           _ptr(mg), b, float(delta), _ptr(out), _ptr(theta_surface),
                                           _ptr(xy_surface), _stream_ptr(stream))
        self._check(st, "fscan_match_batch_polar")
        return out

    def match_host(self, f: np.ndarray, g: np.ndarray, mf=None, mg=None, *, delta: float,
                   surfaces: bool = False):
        """Synchronous batched scan_match on host float32 arrays [B, N, N]."""
        f = np.ascontiguousarray(f, dtype=np.float32)
        g = np.ascontiguousarray(g, dtype=np.float32)
        if f.shape != g.shape or f.ndim not in (2, 3) or f.shape[-1] != self.n or f.shape[-2] != self.n:
            _raise(ERR_INVALID_ARGUMENT, "scan_match: grid specs differ")
        for m in (mf, mg):
            if m is not None and np.shape(m) != f.shape:
                _raise(ERR_INVALID_ARGUMENT, "MaskGrid: shape mismatch")
        if (mf is None) != (mg is None):
            _raise(ERR_INVALID_ARGUMENT, "masks: pass both mask_f and mask_g, or neither")
        if f.ndim == 2:
            f, g = f[None], g[None]
            mf = None if mf is None else np.ascontiguousarray(mf, dtype=np.float32)[None]
            mg = None if mg is None else np.ascontiguousarray(mg, dtype=np.float32)[None]
        mf = None if mf is None else np.ascontiguousarray(mf, dtype=np.float32)
        mg = None if mg is None else np.ascontiguousarray(mg, dtype=np.float32)
        b, n = f.shape[0], f.shape[1]
        if b > self.max_batch:
            _raise(ERR_INVALID_ARGUMENT, f"batch {b} exceeds the context's max_batch {self.max_batch}")
        res = np.zeros(b, dtype=RESULT_DTYPE)
        ts = np.zeros((b, max(1, self.cfg.n_theta)), dtype=np.float64) if surfaces else None
        xs = np.zeros((b, n, n), dtype=np.float32) if surfaces else None
        p = lambda a: None if a is None else a.ctypes.data  # noqa: E731
        st = lib().fscan_match_batch_host(self._h, p(f), p(g), p(mf), p(mg), b, float(delta), p(res), p(ts),
                                          p(xs))
        self._check(st, "fscan_match_batch_host")
        return (res, ts, xs) if surfaces else res

    def estimate_rotation(self, f, g, *, theta=None, theta_surface=None, stream=None):
        f, g = _as_tensor(f), _as_tensor(g)
        import torch
        b = int(f.shape[0])
        self._check_pairs(b, f=f, g=g)
        if theta is None:
            theta = torch.empty(b, dtype=torch.float64, device=f.device)
        _check_tensor(theta, "theta", (b,), "float64")
        _check_bytes(theta_surface, "theta_surface", b * max(1, self.cfg.n_theta) * 8)
        st = lib().fscan_estimate_rotation_batch(self._h, _ptr(f), _ptr(g), b, _ptr(theta), _ptr(theta_surface),
                                                 _stream_ptr(stream))
        self._check(st, "fscan_estimate_rotation_batch")
        return theta

    def estimate_translation(self, f, g, theta, *, delta: float, xy_surface=None, stream=None):
        f, g, theta = _as_tensor(f), _as_tensor(g), _as_tensor(theta)
        import torch
        b = int(f.shape[0])
        self._check_pairs(b, f=f, g=g)
        _check_tensor(theta, "theta", (b,), "float64")
        if xy_surface is not None:
            _check_tensor(xy_surface, "xy_surface", (b, self.n, self.n))
        txy = torch.empty((b, 2), dtype=torch.float64, device=f.device)
        st = lib().fscan_estimate_translation_batch(self._h, _ptr(f), _ptr(g), b, float(delta), _ptr(theta),
                                                    _ptr(txy), _ptr(xy_surface), _stream_ptr(stream))
        self._check(st, "fscan_estimate_translation_batch")
        return txy

    def odometry(self, scans, masks=None, *, delta: float, out=None, theta_surface=None, xy_surface=None,
                 stream=None):
        """Pairs (scan k, scan k+1) of a CUDA sequence [S, N, N] (masks per scan or None):
        S-1 result records, each scan's rotation spectrum computed once."""
        scans, masks = _as_tensor(scans), _as_tensor(masks)
        import torch
        s = int(scans.shape[0])
        _check_tensor(scans, "scans", (s, self.n, self.n))
        _check_tensor(masks, "masks", (s, self.n, self.n))
        if s - 1 > self.max_batch:
            raise ValueError(f"{s - 1} pairs exceed the context's max_batch {self.max_batch}")
        if out is None:
            out = torch.empty(max(s - 1, 0) * RESULT_DTYPE.itemsize, dtype=torch.uint8, device=scans.device)
        self._check_outputs(max(s - 1, 0), out, theta_surface, xy_surface)
        st = lib().fscan_odometry_batch(self._h, _ptr(scans), _ptr(masks), s, float(delta), _ptr(out),
                                        _ptr(theta_surface), _ptr(xy_surface), _stream_ptr(stream))
        self._check(st, "fscan_odometry_batch")
        return out

    def brute_force(self, f, g, thetas, *, delta: float, out=None, stream=None):
        """Exhaustive search over the theta candidates (oracle.cpp:40-67) for a batch
        of CUDA pairs [B, N, N]; returns a uint8 device buffer of BF_DTYPE records
        (decode with decode_bf_results)."""
        f, g = _as_tensor(f), _as_tensor(g)
        import torch
        b = int(f.shape[0])
        self._check_pairs(b, f=f, g=g)
        th = np.ascontiguousarray(np.asarray(thetas, dtype=np.float64).ravel())
        if out is None:
            out = torch.empty(b * BF_DTYPE.itemsize, dtype=torch.uint8, device=f.device)
        _check_bytes(out, "out", b * BF_DTYPE.itemsize)
        st = lib().fscan_brute_force_batch(self._h, _ptr(f), _ptr(g), b, th.ctypes.data, int(th.size),
                                           float(delta), _ptr(out), _stream_ptr(stream))
        self._check(st, "fscan_brute_force_batch")
        return out

    def band_magnitude(self, img, *, stream=None):
        img = _as_tensor(img)
        import torch
        b, n = int(img.shape[0]), int(img.shape[1])
        self._check_pairs(b, img=img)
        out = torch.empty((b, n, n - n // 2), dtype=torch.float32, device=img.device)  # u >= 0 half plane
        st = lib().fscan_band_magnitude_batch(self._h, _ptr(img), b, _ptr(out), _stream_ptr(stream))
        self._check(st, "fscan_band_magnitude_batch")
        return out


def decode_results(buf) -> np.ndarray:
    """uint8 tensor/array of results -> numpy structured array (RESULT_DTYPE)."""
    a = buf.cpu().numpy() if hasattr(buf, "cpu") else np.asarray(buf)
    return np.frombuffer(a.tobytes(), dtype=RESULT_DTYPE).copy()


def decode_bf_results(buf) -> np.ndarray:
    """uint8 tensor/array of brute-force results -> numpy structured array (BF_DTYPE)."""
    a = buf.cpu().numpy() if hasattr(buf, "cpu") else np.asarray(buf)
    return np.frombuffer(a.tobytes(), dtype=BF_DTYPE).copy()


def polar_to_cart(polar, *, range_res: float, n: int, delta: float, stream=None):
    """K0 on CUDA tensors: [B, n_az, n_range] -> [B, n, n] float32."""
    import torch
    b, n_az, n_range = (int(x) for x in polar.shape)
    out = torch.empty((b, n, n), dtype=torch.float32, device=polar.device)
    st = lib().fscan_polar_to_cart_batch(_ptr(polar), b, n_az, n_range, float(range_res), int(n), float(delta),
                                         _ptr(out), _stream_ptr(stream))
    if st != OK:
        _raise(st, "fscan_polar_to_cart_batch")
    return out


# ---------------------------------------------------------------- reference-style single-pair API

@dataclass
class Pose2D:
    theta: float = 0.0
    tx: float = 0.0
    ty: float = 0.0


@dataclass
class MatchResult:
    """Mirror of the pybind11 MatchResult (module.cpp:98-115)."""
    pose: Pose2D
    theta_scores: np.ndarray = field(repr=False)
    theta_coords: np.ndarray = field(repr=False)
    xy_scores: np.ndarray = field(repr=False)
    raw: np.void = field(repr=False, default=None)


_ctx_cache: dict = {}


def scan_match(f, g, delta: float, config: MatchConfig | None = None, mask_f=None, mask_g=None) -> MatchResult:
    """fscan.scan_match(f, g, delta, config) of proj/python/module.cpp:117-136.

    f, g: N x N arrays (any float dtype; converted to float32 for the GPU).
    Without a config, the stock config with the grid geometry swapped in.
    """
    f = np.asarray(f)
    if f.ndim != 2 or f.shape[0] != f.shape[1]:
        _raise(ERR_INVALID_ARGUMENT, "ScanGrid: expected a square n x n grid")
    if np.shape(g) != f.shape:
        _raise(ERR_INVALID_ARGUMENT, "scan_match: grid specs differ")
    for m in (mask_f, mask_g):
        if m is not None and np.shape(m) != f.shape:
            _raise(ERR_INVALID_ARGUMENT, "MaskGrid: shape mismatch")
    n = int(f.shape[0])
    if config is None:
        config = MatchConfig(n_xy=n, delta_xy=delta, n_radius=0)
    cfg = MatchConfig(**config.__dict__).finalize()
    cfg.validate()
    if n != cfg.n_xy:
        _raise(ERR_INVALID_ARGUMENT, "estimate_rotation: grid size != config n_xy")
    key = (tuple(cfg.__dict__.items()),)
    m = _ctx_cache.get(key)
    if m is None:
        m = _ctx_cache[key] = Matcher(cfg, max_batch=1)
    res, ts, xs = m.match_host(f, g, mask_f, mask_g, delta=delta, surfaces=True)
    r = res[0]
    coords = np.array([(k - cfg.n_theta // 2) * cfg.delta_theta for k in range(cfg.n_theta)]) \
        if cfg.n_theta > 1 else np.zeros(1)
    return MatchResult(Pose2D(float(r["theta"]), float(r["tx"]), float(r["ty"])), ts[0][:, None], coords,
                       xs[0].astype(np.float64), r)


def compose(a: Pose2D, b: Pose2D) -> Pose2D:
    """geometry.cpp compose: a then b (b expressed in a's frame)."""
    c, s = math.cos(a.theta), math.sin(a.theta)
    return Pose2D(_normalize_angle(a.theta + b.theta), a.tx + c * b.tx - s * b.ty, a.ty + s * b.tx + c * b.ty)


def inverse(p: Pose2D) -> Pose2D:
    c, s = math.cos(p.theta), math.sin(p.theta)
    return Pose2D(_normalize_angle(-p.theta), -(c * p.tx + s * p.ty), -(-s * p.tx + c * p.ty))


def _normalize_angle(t: float) -> float:
    t = math.fmod(t, 2 * math.pi)
    if t <= -math.pi:
        t += 2 * math.pi
    if t > math.pi:
        t -= 2 * math.pi
    return t


def odometry(scans, delta: float, config: MatchConfig | None = None, masks=None):
    """The odometry command's matching loop (tools/main.cpp:124-135) on the GPU:
    scans [S, N, N] (numpy) -> (absolute poses [S] starting at the identity,
    per-pair result records). rel[k] = inverse(scan_match(scan k, scan k+1).pose)."""
    import torch
    scans = np.ascontiguousarray(scans, dtype=np.float32)
    n_s, n = int(scans.shape[0]), int(scans.shape[1])
    cfg = MatchConfig(**(config or MatchConfig(n_xy=n, delta_xy=delta, n_radius=0)).__dict__).finalize()
    cfg.validate()
    m = Matcher(cfg, max_batch=max(1, n_s - 1))
    dev = torch.device("cuda", m.device)
    s_d = torch.from_numpy(scans).to(dev)
    m_d = None if masks is None else torch.from_numpy(np.ascontiguousarray(masks, dtype=np.float32)).to(dev)
    res = decode_results(m.odometry(s_d, m_d, delta=delta))
    bad = np.nonzero(res["status"] != OK)[0]
    if bad.size:
        _raise(int(res["status"][bad[0]]), f"odometry: pair {int(bad[0])} rejected")
    poses = [Pose2D()]
    for r in res:
        poses.append(compose(poses[-1], inverse(Pose2D(float(r["theta"]), float(r["tx"]), float(r["ty"])))))
    return poses, res


@dataclass
class OracleResult:
    """Mirror of fscan::OracleResult (oracle.hpp:10-13)."""
    pose: Pose2D
    score: float
    raw: np.void = field(repr=False, default=None)


def brute_force_match(f, g, thetas, delta: float, config: MatchConfig | None = None) -> OracleResult:
    """fscan::brute_force_match (oracle.hpp:20-23) for one pair of N x N arrays on the GPU."""
    import torch
    f = np.asarray(f)
    n = int(f.shape[0])
    if np.asarray(g).shape != f.shape:
        _raise(ERR_INVALID_ARGUMENT, "brute_force_match: grid specs differ")
    if len(np.atleast_1d(thetas)) == 0:
        _raise(ERR_INVALID_ARGUMENT, "brute_force_match: empty theta candidate list")
    cfg = MatchConfig(**(config or MatchConfig(n_xy=n, delta_xy=delta, n_radius=0)).__dict__)
    cfg.n_xy = n
    cfg = cfg.finalize()
    key = ("bf", tuple(cfg.__dict__.items()))
    m = _ctx_cache.get(key)
    if m is None:
        m = _ctx_cache[key] = Matcher(cfg, max_batch=1)
    dev = torch.device("cuda", m.device)
    ft = torch.as_tensor(np.ascontiguousarray(f, dtype=np.float32)).to(dev)[None]
    gt = torch.as_tensor(np.ascontiguousarray(g, dtype=np.float32)).to(dev)[None]
    r = decode_bf_results(m.brute_force(ft, gt, thetas, delta=delta))[0]
    return OracleResult(Pose2D(float(r["theta"]), float(r["tx"]), float(r["ty"])), float(r["score"]), r)


# ---------------------------------------------------------------- scan files (.fscn)

def write_scan(path: str, grid, delta: float) -> None:
    """write_scan of proj/src/io.cpp:84-101 (float32 payload)."""
    g = np.ascontiguousarray(grid, dtype=np.float32)
    err = C.create_string_buffer(512)
    st = lib().fscan_fscn_write(os.fsencode(path), g.ctypes.data, int(g.shape[0]), float(delta), err, 512)
    if st != OK:
        _raise(st, err.value.decode() or f"{path}: write failed")


def read_scans(paths, *, threads: int = 0, pinned: bool = False):
    """Read .fscn files (all one grid size) concurrently into one float32 buffer:
    ([B, N, N] numpy array, or a pinned torch tensor for fast H2D, deltas [B])."""
    paths = [os.fsencode(p) for p in paths]
    if not paths:
        return np.zeros((0, 0, 0), np.float32), np.zeros(0)
    n, delta, err = C.c_int(), C.c_double(), C.create_string_buffer(1024)
    st = lib().fscan_fscn_read_header(paths[0], C.byref(n), C.byref(delta), err, 1024)
    if st != OK:
        _raise(st, err.value.decode())
    shape = (len(paths), n.value, n.value)
    if pinned:
        import torch
        buf = torch.empty(shape, dtype=torch.float32, pin_memory=True)
        ptr = buf.data_ptr()
    else:
        buf = np.empty(shape, np.float32)
        ptr = buf.ctypes.data
    deltas = np.empty(len(paths), np.float64)
    arr = (C.c_char_p * len(paths))(*paths)
    st = lib().fscan_fscn_read_batch(arr, len(paths), n.value, ptr, deltas.ctypes.data, int(threads), err, 1024)
    if st != OK:
        _raise(st, err.value.decode())
    return buf, deltas


def odometry_files(paths, config: MatchConfig | None = None):
    """The odometry command's ingestion + matching (tools/main.cpp:104-135): sorted
    .fscn paths -> (absolute poses, per-pair records). Files are read in parallel
    into pinned memory and copied to the device once."""
    import torch
    paths = sorted(paths)
    if len(paths) < 2:
        _raise(ERR_INVALID_ARGUMENT, f"odometry: need at least 2 scans, found {len(paths)}")
    buf, deltas = read_scans(paths, pinned=True)
    n, delta = int(buf.shape[1]), float(deltas[0])
    cfg = MatchConfig(**(config or MatchConfig(n_xy=n, delta_xy=delta, n_radius=0)).__dict__).finalize()
    cfg.validate()
    m = Matcher(cfg, max_batch=len(paths) - 1)
    scans = buf.to(torch.device("cuda", m.device), non_blocking=True)
    res = decode_results(m.odometry(scans, None, delta=delta))
    bad = np.nonzero(res["status"] != OK)[0]
    if bad.size:
        _raise(int(res["status"][bad[0]]), f"odometry: pair {int(bad[0])} rejected")
    poses = [Pose2D()]
    for r in res:
        poses.append(compose(poses[-1], inverse(Pose2D(float(r["theta"]), float(r["tx"]), float(r["ty"])))))
    return poses, res


# ---------------------------------------------------------------- synthetic inputs

def synth_spec(config_id: int, **overrides) -> CSynthSpec:
    s = CSynthSpec()
    if lib().fscan_synth_preset(int(config_id), C.byref(s)) != 0:
        raise ValueError(f"unknown config {config_id}")
    for k, v in overrides.items():
        setattr(s, k, v)
    return s


def synth_pairs_host(spec: CSynthSpec, first: int, count: int, threads: int = 0):
    """(f, g, mf, mg, truth) float32 [count, N, N] (+ float64 [count, 3]) on the host."""
    n = spec.n
    f = np.empty((count, n, n), np.float32)
    g = np.empty_like(f)
    mf = np.empty_like(f)
    mg = np.empty_like(f)
    truth = np.empty((count, 3), np.float64)
    st = lib().fscan_synth_pairs_host(C.byref(spec), first, count, f.ctypes.data, g.ctypes.data, mf.ctypes.data,
                                      mg.ctypes.data, truth.ctypes.data, threads)
    if st:
        raise RuntimeError(f"fscan_synth_pairs_host failed ({st})")
    return f, g, mf, mg, truth


def synth_polar_host(spec: CSynthSpec, first: int, count: int, threads: int = 0):
    pf = np.empty((count, spec.n_az, spec.n_range), np.float32)
    pg = np.empty_like(pf)
    truth = np.empty((count, 3), np.float64)
    st = lib().fscan_synth_polar_host(C.byref(spec), first, count, pf.ctypes.data, pg.ctypes.data,
                                      truth.ctypes.data, threads)
    if st:
        raise RuntimeError(f"fscan_synth_polar_host failed ({st})")
    return pf, pg, truth


def synth_pairs_device(spec: CSynthSpec, first: int, count: int, device: int = 0):
    """Device-rendered pairs as CUDA tensors (f, g, mf, mg) and host truth."""
    import torch
    n = spec.n
    dev = torch.device("cuda", device)
    f = torch.empty((count, n, n), dtype=torch.float32, device=dev)
    g = torch.empty_like(f)
    mf = torch.empty_like(f)
    mg = torch.empty_like(f)
    truth = np.empty((count, 3), np.float64)
    torch.cuda.synchronize(dev)
    st = lib().fscan_synth_pairs_device(C.byref(spec), first, count, f.data_ptr(), g.data_ptr(), mf.data_ptr(),
                                        mg.data_ptr(), truth.ctypes.data, torch.cuda.current_stream(dev).cuda_stream)
    if st:
        raise RuntimeError(f"fscan_synth_pairs_device failed ({st})")
    torch.cuda.synchronize(dev)
    return f, g, mf, mg, truth


def synth_sequence_device(spec: CSynthSpec, seq: int, count: int, device: int = 0):
    """Device-rendered scan sequence (odometry workload) as CUDA tensors (scans, masks)
    [count, N, N] and the host absolute poses [count, 3] (fscan_synth.h)."""
    import torch
    n = spec.n
    dev = torch.device("cuda", device)
    scans = torch.empty((count, n, n), dtype=torch.float32, device=dev)
    masks = torch.empty_like(scans)
    truth = np.empty((count, 3), np.float64)
    torch.cuda.synchronize(dev)
    st = lib().fscan_synth_sequence_device(C.byref(spec), seq, count, scans.data_ptr(), masks.data_ptr(),
                                           truth.ctypes.data, torch.cuda.current_stream(dev).cuda_stream)
    if st:
        raise RuntimeError(f"fscan_synth_sequence_device failed ({st})")
    torch.cuda.synchronize(dev)
    return scans, masks, truth


def synth_polar_device(spec: CSynthSpec, first: int, count: int, device: int = 0):
    import torch
    dev = torch.device("cuda", device)
    pf = torch.empty((count, spec.n_az, spec.n_range), dtype=torch.float32, device=dev)
    pg = torch.empty_like(pf)
    truth = np.empty((count, 3), np.float64)
    torch.cuda.synchronize(dev)
    st = lib().fscan_synth_polar_device(C.byref(spec), first, count, pf.data_ptr(), pg.data_ptr(),
                                        truth.ctypes.data, torch.cuda.current_stream(dev).cuda_stream)
    if st:
        raise RuntimeError(f"fscan_synth_polar_device failed ({st})")
    torch.cuda.synchronize(dev)
    return pf, pg, truth
