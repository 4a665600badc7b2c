#!/usr/bin/env python3
"""Throughput bench of the B200 decoupled Fourier pose search (scan-pair registrations/s).

Workload (BASELINE.json configs[3], "C4"): 4096 scan pairs, 512x512 fp32
Cartesian grids produced from raw polar sweeps by the config-3 generator
(device-rendered, then the product K0 kernel), per-pixel sigmoid masks,
720 azimuth bins, soft-argmax T=1. A step = one full pass of the hot path
(rotation + translation search, pose out, poses gathered to rank 0) over the
job's pairs, inputs resident in HBM (16 GiB > 126 MB L2, so no L2 flush is
needed between steps).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 4]

Multi-GPU (torchrun, one rank per GPU): BASELINE's C4 is ONE 4096-pair batch
sharded by pair index, so by default rank r takes pairs shard_range(4096, N, r)
(strong scaling; --weak gives every rank a full batch). There is no collective
on the hot path; the per-pair result rows are gathered to rank 0 inside every
timed step. Timing is CUDA events on the launching stream, barrier +
synchronize on both sides, max over ranks; rank 0 prints one JSON line.

`--impl reference` times the reference's own CPU implementation (oracle/_ref:
the reference sources + FFTW-API shim) on the host cores, on inputs from the
same seeded generator (oracle/libsynth_gen.so) — that process maps no product
library. Its `config` object is the one this arm prints.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "scan-pair registrations/sec (rot+trans search)"
UNIT = "pairs/s"
# (n, n_theta, masks, batch) of BASELINE.json configs 1..5
CONFIGS = {1: (256, 360, False, 1), 2: (256, 360, True, 64), 3: (512, 720, True, 64),
           4: (512, 720, True, 4096), 5: (1024, 1440, True, 1024)}
POLAR_Q = 400 * 3768  # samples per raw polar sweep (C3)


def workload_desc(cid: int) -> str:
    return {
        1: "C1: 1 pair, 256x256 fp32 Cartesian, 360 bins, hard argmax",
        2: "C2: 64 pairs, 256x256 fp32 Cartesian, sigmoid masks, 360 bins, soft-argmax T=1",
        3: "C3: 64 pairs, raw polar 400x3768 -> 512x512 on device, masks, 720 bins, soft-argmax",
        4: "C4: 4096 pairs, 512x512 fp32 Cartesian from the config-3 polar generator, sigmoid masks, "
           "720 azimuth bins, soft-argmax T=1",
        5: "C5: 1024 pairs, 1024x1024 fp32 Cartesian, sigmoid masks, 1440 bins, soft-argmax T=0.5",
    }[cid]


def job_pairs(args, world: int) -> int:
    base = args.pairs or CONFIGS[args.config][3]
    return base * world if args.weak else base


def input_bytes_per_rank(cid: int, per: int) -> int:
    n, _, masks, _ = CONFIGS[cid]
    grids = (2 * POLAR_Q if cid == 3 else 2 * n * n) + (2 * n * n if masks else 0)
    return 4 * grids * per


def job_config(args, world: int) -> dict:
    """The `config` object both arms print (identical for the same command line)."""
    n, nt, masks, _ = CONFIGS[args.config]
    total = job_pairs(args, world)
    per = -(-total // world)
    ib = input_bytes_per_rank(args.config, per)
    l2 = (f"inputs {ib / 2**30:.1f} GiB per rank per step >> 126 MB L2; no flush needed" if ib >= (512 << 20)
          else f"inputs {ib / 2**20:.0f} MiB per rank per step < 4x L2: L2 flushed (a 256 MiB buffer written) between "
               "timed steps, each step timed by its own events")
    return {"workload": workload_desc(args.config), "pairs": total, "n_xy": n, "n_theta": nt, "masks": masks,
            "parallelism": f"dp{world}: pairs sharded by index ({'weak, a full batch per rank' if args.weak else 'strong, one batch split over the ranks'}), "
                           "no collective on the hot path, result rows gathered to rank 0 every step",
            "l2": l2}


def pair_bytes(n: int, n_theta: int, pad: int, masks: bool = True, s_in: float | None = None) -> float:
    """SURVEY.md §8(d) algorithmic bytes per pair of the canonical staged dataflow."""
    P = 2 * n
    HN = n * (n // 2 + 1)
    HP = P * (P // 2 + 1)
    L = n_theta + 2 * pad
    if s_in is None:
        s_in = 8 * n * n
    return s_in + 8 * (1 if masks else 0) * n * n + 16 * n * n + 16 * HN + 32 * HP + 8 * L + 16


def kernel_alg_bytes(name: str, n: int, wcols: int, masks: bool = True) -> float:
    """Compulsory DRAM bytes per pair of each of OUR kernels.
    wcols = spectrum columns u < W the rotation stage keeps (fscan_ctx_rot_columns):
    K1a stores 2W - 1 columns of the packed spectrum, K1b writes W columns of the
    two magnitude half planes."""
    nn = n * n
    h1 = 3 * n // 4 + 1  # M/2 + 1 spectral bins of the length M = 3N/2 translation transforms
    zc = 2 * wcols - 1
    return {
        "rot_rows": (16 if masks else 8) * nn + 8 * nn + 8 * n * zc,  # f,g(,mf,mg) in; f~,g~ out; Z columns out
        "rot_cols": 8 * n * zc + 8 * n * wcols,           # Z columns in; |F|,|G| (W columns) out
        "rot_gather": 8 * n * wcols,                      # magnitude planes in (polar gather; upper bound)
        "rot_polar": 0.0,                                 # profiles only (fp64 correlation)
        "xlat_rows": 8 * nn + 16 * n * h1,                # f~,g~ in; row spectra (F,G; M/2+1 bins) out
        "xlat_cols": 16 * n * h1 + 8 * n * h1,            # row spectra in; Y (N lags x M/2+1) out
        # Y in; surface out, except in the two-pass form (N >= 512 without requested
        # surfaces: block maxima, then xlat_win recomputes the soft-argmax window rows)
        "xlat_out": 8 * n * h1 + (0 if n >= 512 else 4 * nn),
        "xlat_win": 0.0,                                  # a few Y row blocks per pair (< 8% of xlat_out)
        "finalize": 0.0, "theta_in": 0.0, "mag_unpack": 0.0, "bf_items": 0.0, "bf_final": 0.0,
        "polar_to_cart": 2 * (4 * POLAR_Q + 4 * nn),      # both raw sweeps in, both grids out
    }[name]


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------- helpers

def peaks() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


NCU_TRAFFIC = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def ncu_traffic(kernel: str, n: int) -> float | None:
    """DRAM bytes per pair of `kernel` from the committed ncu --set full capture of a
    C4 chunk (profiles/ncu_traffic.json; None for other grid sides)."""
    try:
        with open(NCU_TRAFFIC) as fh:
            d = json.load(fh)
        if d.get("n_xy", 512) != n:
            return None
        return d.get(kernel, {}).get("dram_bytes_per_pair")
    except Exception:
        return None


def ncu_issue(kernel: str, n: int) -> dict | None:
    """What bounds `kernel` when DRAM does not: its issue-slot and DRAM utilisation in
    the same committed capture (None for a kernel or grid side it did not capture)."""
    try:
        with open(NCU_TRAFFIC) as fh:
            d = json.load(fh)
        if d.get("n_xy", 512) != n or kernel not in d or "issue_pct" not in d[kernel]:
            return None
        k = d[kernel]
        out = {"issue_active_frac": round(k["issue_pct"] / 100, 3), "dram_frac": round(k["dram_pct"] / 100, 3),
               "warps_active_frac": round(k["warps_active_pct"] / 100, 3)}
        # the translation kernels are bound by the L1 data pipe (shared-memory
        # exchanges + loads) before the FMA pipe or DRAM
        for key, name in (("l1_lsu_pct", "l1_lsu_wavefront_frac"), ("fma_pct", "fma_pipe_frac")):
            if key in k:
                out[name] = round(k[key] / 100, 3)
        out["source"] = d.get("source", NCU_TRAFFIC)
        return out
    except Exception:
        return None


def dist_setup(backend: str):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(world, x: float, device) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=device if on_dev else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def loaded_libraries() -> list[str]:
    """Repo .so files mapped into this process (what ran, for the record)."""
    libs = set()
    try:
        with open("/proc/self/maps") as fh:
            for line in fh:
                p = line.split()[-1] if line.strip() else ""
                if p.endswith(".so") and p.startswith(ROOT):
                    libs.add(os.path.relpath(p, ROOT))
    except OSError:
        pass
    return sorted(libs)


def file_sha16(path: str) -> str | None:
    try:
        with open(path, "rb") as fh:
            return hashlib.sha256(fh.read()).hexdigest()[:16]
    except OSError:
        return None


def pct(xs, q):
    xs = sorted(xs)
    if not xs:
        return None
    k = min(len(xs) - 1, max(0, int(math.ceil(q / 100.0 * len(xs))) - 1))
    return xs[k]


def ref_batch(f, g, mf, mg, oc, delta, threads):
    """The reference's own scan_match over a batch (oracle/_ref, parallel_for):
    (seconds, kind, per-pair FoResult array)."""
    import oracle
    if oracle.have_ref():
        t0 = time.perf_counter()
        res = oracle.ref_batch_f32(f, g, mf, mg, oc, delta, threads)
        return time.perf_counter() - t0, "reference", res
    t0 = time.perf_counter()  # the fp64 restatement (port), one pair at a time
    res = [oracle.scan_match(f[i], g[i], oc, delta, None if mf is None else mf[i], None if mg is None else mg[i])
           for i in range(f.shape[0])]
    return time.perf_counter() - t0, "port", res


def cpu_single_thread(f, g, mf, mg, oc, delta, budget_s: float = 6.0) -> dict:
    """Reference scan_match on ONE thread, pair by pair (median / p95 ms per pair)."""
    times = []
    kind = "reference"
    t_end = time.perf_counter() + budget_s
    for i in range(f.shape[0]):
        s, kind, _ = ref_batch(f[i:i + 1], g[i:i + 1], None if mf is None else mf[i:i + 1],
                               None if mg is None else mg[i:i + 1], oc, delta, 1)
        times.append(s * 1e3)
        if time.perf_counter() > t_end and len(times) >= 2:
            break
    return {"value": round(1e3 / statistics.mean(times), 4), "unit": UNIT, "cores": 1, "kind": kind,
            "ms_per_pair_median": round(statistics.median(times), 1), "ms_per_pair_p95": round(pct(times, 95), 1),
            "sample": f"first {len(times)} pairs, one at a time on one thread"}


# ---------------------------------------------------------------- parity (GPU vs the reference, same inputs)

SURF_NEAR_TIE = 4 * 4e-7  # 4x the largest surface error |GPU - oracle| / max|ref| seen in the parity suite


def parity_block(f, g, mf, mg, gpu_rows, ref_rows, oc, delta, kind) -> dict:
    """Integer bins / cells and soft poses of the GPU rows against the reference's own
    scan_match on the same (device-rendered) inputs (BASELINE north_star gates). A
    mismatched bin counts as a documented near-tie only if the reference's top-2 gap
    on that surface is below SURF_NEAR_TIE (SURVEY.md §8(d) rule)."""
    import oracle
    cnt = len(ref_rows)
    tb = np.array([r.theta_bin for r in ref_rows])
    cells = np.array([(r.xy_row, r.xy_col) for r in ref_rows])
    rpose = np.array([(r.theta, r.tx, r.ty) for r in ref_rows])
    gb = gpu_rows["theta_bin"][:cnt]
    gc = np.stack([gpu_rows["xy_row"][:cnt], gpu_rows["xy_col"][:cnt]], 1)
    gpose = np.stack([gpu_rows["theta"][:cnt], gpu_rows["tx"][:cnt], gpu_rows["ty"][:cnt]], 1)
    bins_eq = gb == tb
    cells_eq = (gc == cells).all(1)
    ok = bins_eq & cells_eq
    near, unexplained = [], []
    for i in np.nonzero(~ok)[0][:8]:  # surfaces of the (rare) mismatches, both sides
        r = oracle.scan_match(f[i], g[i], oc, delta, mf[i], mg[i], which="ref" if kind == "reference" else "oracle")
        ts = r.theta_surface
        xs = r.xy_surface
        gap_t = (ts[r.theta_bin] - ts[int(gb[i])]) / np.abs(ts).max()
        gap_x = (xs[r.xy_row, r.xy_col] - xs[int(gc[i][0]), int(gc[i][1])]) / np.abs(xs).max()
        (near if max(gap_t, gap_x) < SURF_NEAR_TIE else unexplained).append(
            {"pair": int(i), "theta_gap": float(gap_t), "xy_gap": float(gap_x)})
    unexplained += [{"pair": int(i)} for i in np.nonzero(~ok)[0][8:]]
    d = np.abs(gpose[ok] - rpose[ok]) if ok.any() else np.zeros((0, 3))
    return {"pairs": int(cnt), "bins_equal": int(bins_eq.sum()), "cells_equal": int(cells_eq.sum()),
            "near_ties": near, "unexplained": unexplained,
            "max_dtheta_rad": float(d[:, 0].max()) if len(d) else None,
            "max_dt_px": float(d[:, 1:].max() / delta) if len(d) else None,
            "gates": {"theta_rad": 1e-3, "t_px": 1e-2},
            "pass": bool(not unexplained and (not len(d) or (d[:, 0].max() <= 1e-3 and d[:, 1:].max() <= 1e-2 * delta))),
            "reference": ("oracle/_ref: the reference's own scan_match (FFTW-API shim)" if kind == "reference"
                          else "fp64 C restatement (oracle/_ref not built)"),
            "inputs": "the GPU run's own device-rendered inputs, copied to the host"}


# ---------------------------------------------------------------- small-batch legs (C1, C2)

def small_config_leg(fb, cid: int, device: int, reps: int) -> dict:
    """BASELINE config `cid` (1: one pair, 2: 64 pairs) timed call by call on this
    GPU: a 256 MiB buffer is written before every call (the inputs would sit in
    L2 otherwise), each call timed by its own events on the launching stream;
    median / p95 per call and pairs/s at the median (the reference's run_bench
    protocol, bench.cpp:53-82: burn-in, then per-call timings)."""
    import torch
    cfg, delta, batch = fb.baseline_config(cid)
    spec = fb.synth_spec(cid)
    f, g, mf, mg, _ = fb.synth_pairs_device(spec, 0, batch, device=device)
    if not spec.masks:
        mf = mg = None
    m = fb.Matcher(cfg, max_batch=batch, device=device)
    m.set_graphs(True)
    dev = torch.device("cuda", device)
    stream = torch.cuda.current_stream(dev)
    out = torch.empty(batch * fb.RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    for _ in range(50):  # burn-in (bench.cpp:56-62)
        m.match_device(f, g, mf, mg, delta=delta, out=out, stream=stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    us = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0.record(stream)
        m.match_device(f, g, mf, mg, delta=delta, out=out, stream=stream)
        e1.record(stream)
        e1.synchronize()
        us.append(e0.elapsed_time(e1) * 1e3)
    res = fb.decode_results(out)
    med = statistics.median(us)
    return {"workload": workload_desc(cid), "value": round(batch / (med / 1e6), 1), "unit": UNIT,
            "us_per_call_median": round(med, 2), "us_per_call_p95": round(pct(us, 95), 2),
            "us_per_pair_median": round(med / batch, 3), "calls": reps, "launches_per_call": m.launches_last,
            "bad_pairs": int((res["status"] != 0).sum()),
            "timing": "per call: L2 flushed before, CUDA events around the graph replay (device time)"}


# ---------------------------------------------------------------- our arm

def run_ours(args):
    import torch
    import paper_2203_00459_b200 as fb
    from paper_2203_00459_b200.shard import gather_results, shard_range

    world, rank, local = dist_setup(args.backend)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg, delta, _ = fb.baseline_config(args.config)
    total = job_pairs(args, world)
    first, per = shard_range(total, world, rank)
    spec = fb.synth_spec(args.config)
    polar = args.config == 3

    # inputs: device-rendered shard (pairs first .. first+per)
    f, g, mf, mg, truth = fb.synth_pairs_device(spec, first, per, device=local)
    if not spec.masks:
        mf = mg = None
    m = fb.Matcher(cfg, max_batch=max(per, 1), device=local, chunk=args.chunk)
    if not args.no_graphs:
        m.set_graphs(True)  # replay the call's launch sequence as one CUDA graph (fscan_ctx_set_graphs)
    out = torch.empty(per * fb.RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    if polar:  # C3: the raw sweeps are the input; K0 runs inside every step
        pf, pg, _ = fb.synth_polar_device(spec, first, per, device=local)

    def step():
        if polar:
            return m.match_polar(pf, pg, mf, mg, range_res=spec.range_res, delta=delta, out=out, stream=stream)
        return m.match_device(f, g, mf, mg, delta=delta, out=out, stream=stream)

    rows = out.view(per, fb.RESULT_DTYPE.itemsize)

    def gather():  # pose gather to rank 0 (inside the timed step)
        return gather_results(rows, total, world, rank)

    for _ in range(args.warmup):
        step()
        gather()
    torch.cuda.synchronize(dev)
    launches_per_step = m.launches_last

    # inputs that fit in the 126 MB L2 (C1/C2) are timed step by step with a 256 MiB
    # buffer written between the steps, outside the events
    flush = None
    if input_bytes_per_rank(args.config, per) < (512 << 20):
        flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    barrier(world)
    torch.cuda.synchronize(dev)
    gathered = None
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            if flush is not None:
                with torch.cuda.stream(stream):
                    flush.fill_(1.0)
            if flush is not None or i == 0:
                evs[2 * i].record(stream)
            step()
            gathered = gather()
            evs[2 * i + 1].record(stream)
        torch.cuda.synchronize(dev)
    if flush is None:  # back to back: step i spans end(i-1) .. end(i)
        ends = [evs[2 * i + 1] for i in range(args.steps)]
        step_ms = [evs[0].elapsed_time(ends[0])] + [ends[i - 1].elapsed_time(ends[i]) for i in range(1, args.steps)]
    else:
        step_ms = [evs[2 * i].elapsed_time(evs[2 * i + 1]) for i in range(args.steps)]
    ms = sum(step_ms)
    barrier(world)
    ms_max = allmax(world, ms, dev)
    value = total * args.steps / (ms_max / 1e3)
    bad = None
    res0 = None
    if rank == 0:
        res0 = fb.decode_results(gathered.reshape(-1))
        bad = int((res0["status"] != 0).sum())
    if args.dump_results and rank == 0:
        np.save(args.dump_results, res0)

    # per-kernel breakdown: one instrumented step (events around every kernel)
    m.set_profiling(True)
    step()
    torch.cuda.synchronize(dev)
    kt = m.kernel_times()
    m.set_profiling(False)
    dom = max(kt.items(), key=lambda kv: kv[1][0])[0]
    dom_ms, dom_launches = kt[dom]
    pairs_per_launch = per / dom_launches
    wcols = m.rot_columns
    alg = kernel_alg_bytes(dom, cfg.n_xy, wcols, mf is not None) * pairs_per_launch
    achieved = alg / (dom_ms / dom_launches / 1e3) / 1e9
    peak, peak_src = peaks()
    traffic = ncu_traffic(dom, cfg.n_xy)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "peak_source": peak_src,
                "traffic": None if traffic is None else traffic * pairs_per_launch,
                "alg_bytes_per_launch": alg, "pairs_per_launch": round(pairs_per_launch, 2),
                "avg_launch_ms": dom_ms / dom_launches,
                "kernel_share": round(dom_ms / sum(v[0] for v in kt.values()), 3),
                # the dominant kernel is bound by its L1 data pipe and issue slots, not
                # by DRAM: its ncu utilisations say how close it runs to those ceilings
                "ncu": ncu_issue(dom, cfg.n_xy)}
    bpair = pair_bytes(cfg.n_xy, cfg.n_theta, cfg.pad_angle, masks=mf is not None,
                       s_in=(8.0 * spec.n_az * spec.n_range) if polar else None)
    pipeline = {"b_pair_bytes": bpair, "achieved_gbs": round(value * bpair / 1e9 / world, 1),
                "frac_of_measured_peak_per_gpu": round(value * bpair / world / (peak * 1e9), 4),
                "frac_of_8TBps_per_gpu": round(value * bpair / world / 8e12, 4),
                "kernel_ms_per_step": {k: round(v[0], 3) for k, v in kt.items()},
                "kernel_alg_gbs": {k: round(kernel_alg_bytes(k, cfg.n_xy, wcols, mf is not None) * per
                                            / (v[0] / 1e3) / 1e9, 1) for k, v in kt.items()
                                   if kernel_alg_bytes(k, cfg.n_xy, wcols, mf is not None) > 0}}

    # per-GPU efficiency at the 4- and 8-GPU shard sizes of this job (1-GPU proxy
    # of the strong-scaling curve before 8-GPU hardware is available)
    proxy = None
    if rank == 0 and world == 1 and not args.no_proxy and not polar and total >= 256:
        proxy = {}
        for shard in sorted({total // 8, total // 4, total // 2}):
            so = torch.empty(shard * fb.RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
            call = lambda: m.match_device(f[:shard], g[:shard], None if mf is None else mf[:shard],  # noqa: E731
                                          None if mg is None else mg[:shard], delta=delta, out=so, stream=stream)
            for _ in range(3):
                call()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(3, args.steps)
            e0.record(stream)
            for _ in range(reps):
                call()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            rate = shard * reps / (e0.elapsed_time(e1) / 1e3)
            proxy[str(shard)] = {"pairs_per_s": round(rate, 1), "per_gpu_efficiency": round(rate / value, 3),
                                 "as_shard_of": f"{total // shard} GPUs"}

    # BASELINE C1 (single-pair latency) and C2 (64-pair batch) measured in the
    # same run (rank 0, N = 1, on the default C4 job)
    small = None
    if rank == 0 and world == 1 and args.config == 4 and not args.no_small:
        small = {"c1": small_config_leg(fb, 1, local, 200), "c2": small_config_leg(fb, 2, local, 100)}

    # the paper's central comparison: the exhaustive correlative search (the
    # reference's brute_force_match, oracle.cpp:40-67) over the matcher's full theta
    # grid on the same GPU, a few pairs (every candidate is one translation stage)
    exhaustive = None
    if rank == 0 and not args.no_exhaustive and not polar:
        nb = min(per, 4)
        thetas = np.array([(k - cfg.n_theta // 2) * cfg.delta_theta for k in range(cfg.n_theta)])
        mb = fb.Matcher(cfg, max_batch=nb, device=local)
        mb.brute_force(f[:nb], g[:nb], thetas, delta=delta, stream=stream)  # warm
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        mb.brute_force(f[:nb], g[:nb], thetas, delta=delta, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        bf_rate = nb / (e0.elapsed_time(e1) / 1e3)
        exhaustive = {"value": round(bf_rate, 2), "unit": UNIT, "candidates": int(cfg.n_theta), "sample_pairs": nb,
                      "decoupled_speedup": round(value / world / bf_rate, 1),
                      "api": "fscan_brute_force_batch (unmasked scans, matcher theta grid)"}
        del mb

    # odometry chaining: the same number of pairs registered as
    # consecutive scans of one sequence, each scan's rotation spectrum shared by its
    # two pairs; reported beside the independent-pair value
    chain = None
    if rank == 0 and not args.no_odometry and not polar and per >= 2:
        seq, seqm, _ = fb.synth_sequence_device(spec, first, per + 1, device=local)
        mo = fb.Matcher(cfg, max_batch=per, device=local, chunk=args.chunk)
        oout = torch.empty(per * fb.RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        mo.odometry(seq, seqm, delta=delta, out=oout, stream=stream)  # warm
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(1, min(args.steps, 5))
        e0.record(stream)
        for _ in range(reps):
            mo.odometry(seq, seqm, delta=delta, out=oout, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        rate = per * reps / (e0.elapsed_time(e1) / 1e3)
        chain = {"value": round(rate, 1), "unit": UNIT, "pairs": per, "steps": reps,
                 "vs_independent_pairs": round(rate / (value / world), 3),
                 "api": "fscan_odometry_batch (scan k vs scan k+1 of a generated drive, masks per scan)"}
        del mo, seq, seqm, oout

    # e2e through the public host API (H2D + compute + D2H each step)
    e2e = None
    if not args.no_e2e and not polar:
        try:
            import psutil
            grids = 4 if mf is not None else 2
            need = grids * f.numel() * 4 * 1.2
            if psutil.virtual_memory().available < need + (8 << 30):
                raise MemoryError("not enough host RAM for pinned inputs")
            hs = [torch.empty(f.shape, dtype=torch.float32, pin_memory=True) for _ in range(grids)]
            for h, d in zip(hs, (f, g, mf, mg)):
                h.copy_(d)
            nps = [h.numpy() for h in hs] + [None] * (4 - grids)
            m.match_host(*nps, delta=delta)  # warm
            steps_e2e = max(1, min(args.steps, 10))
            barrier(world)
            t0 = time.perf_counter()
            for _ in range(steps_e2e):
                m.match_host(*nps, delta=delta)
            dt = allmax(world, time.perf_counter() - t0, dev)
            e2e = {"value": round(total * steps_e2e / dt, 1), "unit": UNIT,
                   "h2d_bytes_per_step": int(grids * f.numel() * 4 * world),
                   "d2h_bytes_per_step": int(total * fb.RESULT_DTYPE.itemsize), "steps": steps_e2e,
                   "api": "fscan_match_batch_host (pinned host buffers)"}
            # what bounds it: this rank's H2D rate inside the e2e steps against a
            # plain pinned -> device copy of one input grid set on the same link
            e2e["h2d_gbs"] = round(grids * f.numel() * 4 * steps_e2e / dt / 1e9, 1)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dst = torch.empty_like(f)
            dst.copy_(hs[0], non_blocking=True)
            torch.cuda.synchronize()
            best = float("inf")
            for _ in range(3):
                c0.record()
                dst.copy_(hs[0], non_blocking=True)
                c1.record()
                c1.synchronize()
                best = min(best, c0.elapsed_time(c1) / 1e3)
            e2e["pinned_copy_h2d_gbs"] = round(hs[0].numel() * 4 / best / 1e9, 1)
            del hs, nps, dst
        except Exception as exc:  # report, never fake
            e2e = {"value": None, "unit": UNIT, "error": str(exc)[:200]}

    # CPU baseline + parity: the reference on the host cores on a bounded sample of
    # this run's own inputs (rank 0, N=1), results compared with the GPU's rows
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu and not polar:
        import oracle
        oc = oracle.make_config(**{k: (int(v) if isinstance(v, bool) else v) for k, v in cfg.__dict__.items()})
        threads = cpu_threads()
        # pilot of one pair per thread, then a sample sized for ~12 s of CPU work
        pilot = int(min(per, threads))
        host = lambda k: [None if x is None else x[:k].cpu().numpy() for x in (f, g, mf, mg)]  # noqa: E731
        psecs, _, _ = ref_batch(*host(pilot), oc, delta, threads)
        sample = int(min(per, max(pilot, round(12.0 * pilot / max(psecs, 1e-3) / threads) * threads)))
        hs = host(sample)
        secs, kind, ref_rows = ref_batch(*hs, oc, delta, threads)
        cpu = {"value": round(sample / secs, 3), "unit": UNIT, "cores": threads, "kind": kind,
               "sample": f"first {sample} pairs of the {workload_desc(args.config).split(':')[0]} workload "
                         f"({secs:.1f} s wall, reference scan_match via parallel_for, FFTW-API shim not FFTW)",
               "single_thread": cpu_single_thread(*hs, oc, delta),
               "host": oracle.host_descriptor()}
        gpu_rows = fb.decode_results(out)
        parity = parity_block(*hs, gpu_rows, ref_rows, oc, delta, kind)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3),
            "step_ms": {"median": round(statistics.median(step_ms), 3), "p95": round(pct(step_ms, 95), 3),
                        "min": round(min(step_ms), 3)},
            "higher_is_better": True, "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (seeded generator)",
            "config": job_config(args, world),
            "impl_config": {"chunk": args.chunk or "auto", "graphs": not args.no_graphs,
                            "pairs_per_rank": per, "backend": args.backend if world > 1 else None},
            "roofline": roofline, "hbm_pipeline": pipeline, "cpu_baseline": cpu, "parity": parity,
            "e2e": e2e, "shard_proxy": proxy, "small_batches": small, "exhaustive_search": exhaustive,
            "odometry_chain": chain,
            "clocks": clk.summary(), "gpu_launches": launches_per_step * args.steps,
            "bad_pairs": bad, "impl": "ours",
            "library": {"path": os.path.relpath(fb.LIB_PATH, ROOT), "sha16": file_sha16(fb.LIB_PATH),
                        "loaded": loaded_libraries()},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------- reference arm

def run_reference(args):
    """The reference's own CPU scan_match (oracle/_ref) on the host cores: every step a
    bounded sample of the job (one pair per host thread), inputs from the same seeded
    generator (oracle/libsynth_gen.so). Maps no product library."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oc, delta, _ = oracle.baseline_config(args.config)
    threads = cpu_threads()
    sample = threads
    if args.config == 1:
        sample = 1
    f, g, mf, mg, _ = oracle.synth_pairs_host(args.config, 0, sample, threads=threads)
    if not CONFIGS[args.config][2]:
        mf = mg = None
    for _ in range(args.warmup):
        ref_batch(f, g, mf, mg, oc, delta, threads)
    secs = []
    kind = "reference"
    for _ in range(args.steps):
        s, kind, _ = ref_batch(f, g, mf, mg, oc, delta, threads)
        secs.append(s)
    tot = sum(secs)
    value = sample * args.steps / tot
    single = cpu_single_thread(f, g, mf, mg, oc, delta, budget_s=5.0)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * tot / args.steps, 1),
        "step_ms": {"median": round(1e3 * statistics.median(secs), 1), "p95": round(1e3 * pct(secs, 95), 1),
                    "min": round(1e3 * min(secs), 1)},
        "higher_is_better": True, "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generator)",
        "config": job_config(args, world),
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{sample} pairs of the job per step (pairs 0..{sample - 1}, one per host "
                                   f"thread), reference scan_match via parallel_for on {threads} threads "
                                   "(FFTW-API shim, not FFTW)",
                         "single_thread": single, "host": oracle.host_descriptor()},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "library": {"loaded": loaded_libraries()},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=4, choices=(1, 2, 3, 4, 5))
    ap.add_argument("--pairs", type=int, default=0, help="override the config's pair count")
    ap.add_argument("--chunk", type=int, default=0, help="pairs per pipeline chunk (0 = auto)")
    ap.add_argument("--no-graphs", action="store_true", help="launch the kernels directly instead of "
                    "replaying the match call's CUDA graph")
    ap.add_argument("--weak", action="store_true",
                    help="every rank registers a full batch (default: the batch is split over the ranks)")
    ap.add_argument("--backend", choices=("nccl", "gloo"), default="nccl",
                    help="torch.distributed backend for N > 1 (gloo: the CPU-side test of the multi-rank path)")
    ap.add_argument("--dump-results", default="", help="rank 0 saves the gathered result rows (.npy)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-proxy", action="store_true", help="skip the per-shard-size proxy lines")
    ap.add_argument("--no-small", action="store_true", help="skip the C1 latency / C2 batch legs")
    ap.add_argument("--no-exhaustive", action="store_true", help="skip the brute-force comparison leg")
    ap.add_argument("--no-odometry", action="store_true", help="skip the chained-sequence leg")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
