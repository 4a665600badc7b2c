#!/usr/bin/env python3
"""Throughput bench of the B200 decoupled Fourier pose search (scan-pair registrations/s).

Workload (BASELINE.json configs[3], "C4"): 4096 scan pairs, 512x512 fp32
Cartesian grids produced from raw polar sweeps by the config-3 generator
(device-rendered, then the product K0 kernel), per-pixel sigmoid masks,
720 azimuth bins, soft-argmax T=1, sharded by pair index over the ranks.
A step = one full pass of the hot path (rotation + translation search, pose
out) over the rank's shard, inputs resident in HBM (16 GiB > 126 MB L2, so no
L2 flush is needed between steps).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 4]

Under torchrun each rank takes pairs [r*B/N, (r+1)*B/N); timing is CUDA
events on the launching stream, barrier + synchronize on both sides, max over
ranks; rank 0 prints one JSON line. `--impl reference` times the reference's
own CPU implementation (oracle/_ref: the reference sources + FFTW-API shim)
on the host cores instead (rank 0 only).
"""
from __future__ import annotations

import argparse
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
KERNEL_NAMES = ("rot_rows", "rot_cols", "rot_polar", "theta_in", "xlat_rows", "xlat_cols", "xlat_out",
                "finalize", "rot_gather", "polar_to_cart", "mag_unpack", "bf_items", "bf_final")


def workload_desc(cid: int) -> str:
    return {
        1: "C1: 1 pair, 256x256 fp32 Cartesian, 360 bins, hard argmax",
        2: "C2: 64 pairs, 256x256 fp32 Cartesian, sigmoid masks, 360 bins, soft-argmax T=1",
        3: "C3: 64 pairs, raw polar 400x3768 -> 512x512 on device, masks, 720 bins, soft-argmax",
        4: "C4: 4096 pairs, 512x512 fp32 Cartesian from the config-3 polar generator, sigmoid masks, "
           "720 azimuth bins, soft-argmax T=1",
        5: "C5: 1024 pairs, 1024x1024 fp32 Cartesian, sigmoid masks, 1440 bins, soft-argmax T=0.5",
    }[cid]


def pair_bytes(n: int, n_theta: int, pad: int, masks: bool = True, s_in: float | None = None) -> float:
    """SURVEY.md §8(d) algorithmic bytes per pair of the canonical staged dataflow."""
    P = 2 * n
    HN = n * (n // 2 + 1)
    HP = P * (P // 2 + 1)
    L = n_theta + 2 * pad
    if s_in is None:
        s_in = 8 * n * n
    return s_in + 8 * (1 if masks else 0) * n * n + 16 * n * n + 16 * HN + 32 * HP + 8 * L + 16


def kernel_alg_bytes(name: str, n: int) -> float:
    """Compulsory DRAM bytes per pair of each of OUR kernels."""
    nn = n * n
    h1 = 3 * n // 4 + 1  # M/2 + 1 spectral bins of the length M = 3N/2 translation transforms
    return {
        "rot_rows": 16 * nn + 8 * nn + 8 * nn,            # f,g,mf,mg in; f~,g~ out; Z out
        "rot_cols": 8 * nn + 4 * nn,                      # Z in; |F|,|G| half planes out
        "rot_gather": 4 * nn,                             # magnitude planes in (polar gather)
        "rot_polar": 0.0,                                 # profiles only (fp64 correlation)
        "xlat_rows": 8 * nn + 16 * n * h1,                # f~,g~ in; row spectra (F,G; M/2+1 bins) out
        "xlat_cols": 16 * n * h1 + 8 * n * h1,            # row spectra in; Y (N lags x M/2+1) out
        "xlat_out": 8 * n * h1 + 4 * nn,                  # Y in; surface out
        "finalize": 0.0,
        "theta_in": 0.0,
        "mag_unpack": 0.0,
        "bf_items": 0.0,
        "bf_final": 0.0,
        "polar_to_cart": 2 * (4 * 400 * 3768 + 4 * nn),   # both raw sweeps in, both grids out
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
            self._stop.wait(0.2)

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


def ncu_traffic(kernel: str) -> float | None:
    """DRAM bytes per launch of `kernel` from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get(kernel, {}).get("dram_bytes_per_pair")
    except Exception:
        return None


def ncu_issue(kernel: str, n: int) -> dict | None:
    """What bounds `kernel` when DRAM does not: its issue-slot and DRAM utilisation
    in the committed ncu --set full capture (profiles/r01/ncu_full_summary.json,
    the C4 grid side; None for a kernel or grid side it did not capture)."""
    path = os.path.join(ROOT, "profiles", "r01", "ncu_full_summary.json")
    try:
        with open(path) as fh:
            for k in json.load(fh)["kernels"]:
                if n != 512:  # the capture is of one C4 chunk (N = 512)
                    return None
                if k["kernel"].partition("<")[0] == "k_" + kernel:
                    return {"issue_active_frac": round(k["issue_pct"] / 100, 3),
                            "dram_frac": round(k["dram_pct"] / 100, 3),
                            "source": "ncu --set full, profiles/r01/ncu_full_summary.json"}
    except Exception:
        return None
    return None


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
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
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def ref_cpu_run(f, g, mf, mg, cfg, delta, threads):
    """The reference's own scan_match over a batch (oracle/_ref, parallel_for)."""
    import oracle
    oc = oracle.make_config(**{k: (int(v) if isinstance(v, bool) else v) for k, v in cfg.__dict__.items()})
    if oracle.have_ref():
        t0 = time.perf_counter()
        oracle.ref_batch_f32(f, g, mf, mg, oc, delta, threads)
        return time.perf_counter() - t0, "reference"
    # port fallback (restatement), single thread per call
    t0 = time.perf_counter()
    for i in range(f.shape[0]):
        oracle.scan_match(f[i], g[i], oc, delta, mf[i], mg[i])
    return time.perf_counter() - t0, "port"


# ---------------------------------------------------------------- our arm

def run_ours(args):
    import torch
    import paper_2203_00459_b200 as fb

    world, rank, local = dist_setup()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg, delta, total = fb.baseline_config(args.config)
    if args.pairs:
        total = args.pairs
    # weak scaling (default): every rank registers the config's batch, a disjoint
    # block of pair indices of a world x batch job; --strong splits one batch
    if not args.strong:
        total *= world
    from paper_2203_00459_b200.shard import gather_results, shard_range
    first, per = shard_range(total, world, rank)
    spec = fb.synth_spec(args.config)

    # inputs: device-rendered shard (pairs first .. first+per)
    f, g, mf, mg, truth = fb.synth_pairs_device(spec, first, per, device=local)
    m = fb.Matcher(cfg, max_batch=per, device=local, chunk=args.chunk)
    if not args.no_graphs:
        m.set_graphs(True)  # replay the call's launch sequence as one CUDA graph (fscan_ctx_set_graphs)
    out = torch.empty(per * fb.RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    polar = args.config == 3
    if polar:  # C3: the raw sweeps are the input; K0 runs inside every step
        pf, pg, _ = fb.synth_polar_device(spec, first, per, device=local)

    def step():
        if polar:
            return m.match_polar(pf, pg, mf, mg, range_res=spec.range_res, delta=delta, out=out, stream=stream)
        return m.match_device(f, g, mf, mg, delta=delta, out=out, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    launches_per_step = m.launches_last
    res = fb.decode_results(out)
    bad = int((res["status"] != 0).sum())

    # inputs that fit in the 126 MB L2 (C2: 64 pairs of 256^2) are timed step by
    # step with a 256 MB buffer written between the steps, outside the events
    in_bytes = sum(t.numel() * t.element_size() for t in ((pf, pg) if polar else (f, g)) + (mf, mg)
                   if t is not None)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev) if in_bytes < (512 << 20) else None
    l2_note = (f"inputs {in_bytes / 2**20:.0f} MiB per step < 2x L2: a 256 MiB buffer written between timed "
               "steps, each step timed by its own events" if flush is not None else
               f"inputs {in_bytes / 2**30:.1f} GiB per step >> 126 MB L2; no flush needed")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        if flush is None:
            ev0.record(stream)
            for _ in range(args.steps):
                step()
            ev1.record(stream)
            torch.cuda.synchronize(dev)
            ms = ev0.elapsed_time(ev1)
        else:
            ms = 0.0
            for _ in range(args.steps):
                with torch.cuda.stream(stream):
                    flush.fill_(1.0)
                ev0.record(stream)
                step()
                ev1.record(stream)
                torch.cuda.synchronize(dev)
                ms += ev0.elapsed_time(ev1)
    barrier(world)
    ms_max = allmax(world, ms, dev)
    value = total * args.steps / (ms_max / 1e3)

    # pose gather to rank 0 (off the timed region): [total, sizeof(result)] bytes in pair order
    rows = out.view(per, fb.RESULT_DTYPE.itemsize)
    gathered = gather_results(rows, total, world, rank)
    if rank == 0:
        allres = fb.decode_results(gathered.reshape(-1))
        bad = int((allres["status"] != 0).sum())

    # per-kernel breakdown: one instrumented step (events around every kernel)
    m.set_profiling(True)
    step()
    torch.cuda.synchronize(dev)
    kt = m.kernel_times()
    m.set_profiling(False)
    dom = max(kt.items(), key=lambda kv: kv[1][0])[0]
    dom_ms, dom_launches = kt[dom]
    pairs_per_launch = per / dom_launches
    alg = kernel_alg_bytes(dom, cfg.n_xy) * pairs_per_launch
    achieved = alg / (dom_ms / dom_launches / 1e3) / 1e9
    peak, peak_src = peaks()
    traffic = ncu_traffic(dom)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "peak_source": peak_src,
                "traffic": None if traffic is None else traffic * pairs_per_launch,
                "alg_bytes_per_launch": alg, "avg_launch_ms": dom_ms / dom_launches,
                "kernel_share": round(dom_ms / sum(v[0] for v in kt.values()), 3),
                # the dominant kernel is FFT-issue-bound, not DRAM-bound: its ncu issue
                # utilisation says how close it runs to its own ceiling
                "ncu": ncu_issue(dom, cfg.n_xy)}
    bpair = pair_bytes(cfg.n_xy, cfg.n_theta, cfg.pad_angle,
                       s_in=(8.0 * spec.n_az * spec.n_range) if polar else None)
    pipeline = {"b_pair_bytes": bpair, "achieved_gbs": round(value * bpair / 1e9 / world, 1),
                "frac_of_measured_peak_per_gpu": round(value * bpair / world / (peak * 1e9), 4),
                "frac_of_8TBps_per_gpu": round(value * bpair / world / 8e12, 4),
                "kernel_ms_per_step": {k: round(v[0], 3) for k, v in kt.items()}}

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
    if rank == 0 and not args.no_odometry and not polar:
        # a generated drive: per + 1 scans of one scene, consecutive scans related
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
    if not args.no_e2e:
        try:
            import psutil
            need = 4 * f.numel() * 4 * 1.2
            if psutil.virtual_memory().available < need + (8 << 30):
                raise MemoryError("not enough host RAM for pinned inputs")
            hf, hg, hmf, hmg = (torch.empty(f.shape, dtype=torch.float32, pin_memory=True) for _ in range(4))
            for h, d in ((hf, f), (hg, g), (hmf, mf), (hmg, mg)):
                h.copy_(d)
            nf, ng, nmf, nmg = (h.numpy() for h in (hf, hg, hmf, hmg))
            m.match_host(nf, ng, nmf, nmg, delta=delta)  # warm
            steps_e2e = max(1, min(args.steps, 3))
            barrier(world)
            t0 = time.perf_counter()
            for _ in range(steps_e2e):
                m.match_host(nf, ng, nmf, nmg, delta=delta)
            dt = allmax(world, time.perf_counter() - t0, dev)
            e2e = {"value": round(total * steps_e2e / dt, 1), "unit": UNIT,
                   "h2d_bytes_per_step": int(4 * f.numel() * 4 * world),
                   "d2h_bytes_per_step": int(total * fb.RESULT_DTYPE.itemsize), "steps": steps_e2e,
                   "api": "fscan_match_batch_host (pinned host buffers)"}
            # what bounds it: this rank's H2D rate inside the e2e steps against a
            # plain pinned -> device copy of one input grid set on the same link
            e2e["h2d_gbs"] = round(4 * f.numel() * 4 * steps_e2e / dt / 1e9, 1)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dst = torch.empty_like(f)
            dst.copy_(hf, non_blocking=True)
            torch.cuda.synchronize()
            best = float("inf")
            for _ in range(3):
                c0.record()
                dst.copy_(hf, non_blocking=True)
                c1.record()
                c1.synchronize()
                best = min(best, c0.elapsed_time(c1) / 1e3)
            e2e["pinned_copy_h2d_gbs"] = round(hf.numel() * 4 / best / 1e9, 1)
            del hf, hg, hmf, hmg, dst
        except Exception as exc:  # report, never fake
            e2e = {"value": None, "unit": UNIT, "error": str(exc)[:200]}

    # CPU baseline: the reference on the host cores, bounded sample (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = cpu_threads()
        # pilot of one pair per thread, then a sample sized for ~15 s of CPU work
        pilot = int(min(per, threads))
        hs = [x[:pilot].cpu().numpy() for x in (f, g, mf, mg)]
        psecs, _ = ref_cpu_run(*hs, cfg, delta, threads)
        sample = int(min(per, max(pilot, round(15.0 * pilot / max(psecs, 1e-3) / threads) * threads)))
        hs = [x[:sample].cpu().numpy() for x in (f, g, mf, mg)]
        secs, kind = ref_cpu_run(*hs, cfg, delta, threads)
        cpu = {"value": round(sample / secs, 3), "unit": UNIT, "cores": threads, "kind": kind,
               "sample": f"first {sample} pairs of the {workload_desc(args.config).split(':')[0]} workload "
                         f"({secs:.1f} s wall, reference scan_match via parallel_for, FFTW-API shim not FFTW)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded generator)",
            "config": {"workload": workload_desc(args.config), "pairs": total, "pairs_per_rank": per,
                       "n_xy": cfg.n_xy, "n_theta": cfg.n_theta, "chunk": args.chunk or "auto",
                       "l2": l2_note, "graphs": not args.no_graphs,
                       "parallelism": f"dp{world} (pairs sharded by index, no collective on the hot path)"},
            "roofline": roofline, "hbm_pipeline": pipeline, "cpu_baseline": cpu, "e2e": e2e,
            "exhaustive_search": exhaustive, "odometry_chain": chain,
            "clocks": clk.summary(), "gpu_launches": launches_per_step * args.steps,
            "bad_pairs": bad, "impl": "ours",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ---------------------------------------------------------------- reference arm

def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import paper_2203_00459_b200 as fb  # config + host generator only (no GPU code runs)
    cfg, delta, total = fb.baseline_config(args.config)
    threads = cpu_threads()
    sample = int(max(8, min(threads, 128)))
    spec = fb.synth_spec(args.config)
    f, g, mf, mg, _ = fb.synth_pairs_host(spec, 0, sample, threads=threads)
    kind = "reference" if oracle.have_ref() else "port"
    for _ in range(args.warmup):
        ref_cpu_run(f[:threads], g[:threads], mf[:threads], mg[:threads], cfg, delta, threads)
    secs = []
    for _ in range(args.steps):
        s, kind = ref_cpu_run(f, g, mf, mg, cfg, delta, threads)
        secs.append(s)
    tot = sum(secs)
    value = sample * args.steps / tot
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * tot / args.steps, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator)",
        "config": {"workload": workload_desc(args.config), "pairs_per_step": sample, "n_xy": cfg.n_xy,
                   "n_theta": cfg.n_theta},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{sample} pairs of the workload per step, reference scan_match via "
                                   f"parallel_for on {threads} threads (FFTW-API shim, not FFTW)"},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-exhaustive", action="store_true", help="skip the brute-force comparison leg")
    ap.add_argument("--no-odometry", action="store_true", help="skip the chained-sequence leg")
    ap.add_argument("--strong", action="store_true",
                    help="split the config's batch over the ranks (default: weak scaling, one batch per rank)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
