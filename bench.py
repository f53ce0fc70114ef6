#!/usr/bin/env python3
"""Benchmark of the B200 dual-domain CSC hot path (BASELINE.json metric).

Default workload (N=1): BASELINE.json configs[1] (C1) — coding subproblem,
dictionary fixed (the generator's ground truth), N=256 images 128x128 FP32,
K=64 filters 11x11, 50 ADMM iterations, beta=0.5, cold start. One step = one
coding outer iteration over all images (solve_coding for every image, the
coding half-step of run_csc, pipeline.cpp:221-227). --config c2/c4/c0 runs the
full coding+learning outer iteration (run_csc) instead.

value  = outer iterations/s with inputs resident in HBM (device events).
e2e    = the same metric through the C-ABI with host buffers each step
         (signals h2d + coding + per-image stats d2h), host wall clock.
Multi-GPU: one process per GPU, max-over-ranks device timing. Coding-only
configs (C1 default) scale weakly: each rank codes its own N-image C1 workload
(images are independent units; no data-path collective), value = world x
steps / time. Full configs (--config c0/c2/c3/c4) split their N images over
the ranks (strong scaling; learning all-reduces its correlations).

--impl reference times the reference's own CPU implementation
(oracle/_ref/libdcsc_ref.so, the unmodified reference solver TUs) on the
box's host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CSC ADMM outer iters/s (coding+learning) at N,K,H×W; % of HBM roofline"
UNIT = "outer_iters/s"

CONFIGS = {
    # name: N, H, W, K, m, precision, beta, p, sigma, coding_only, max_admm, outer
    "c0": dict(N=10, H=100, W=100, K=100, m=11, prec=64, beta=1.0, p=0.01, sigma=0.01, coding_only=False,
               max_admm=500, outer=10),
    "c1": dict(N=256, H=128, W=128, K=64, m=11, prec=32, beta=0.5, p=0.01, sigma=0.01, coding_only=True,
               max_admm=50, outer=1),
    "c2": dict(N=100, H=100, W=100, K=100, m=11, prec=32, beta=0.5, p=0.02, sigma=0.01, coding_only=False,
               max_admm=500, outer=20),
    "c3": dict(N=512, H=256, W=256, K=128, m=11, prec=32, beta=0.5, p=0.01, sigma=0.01, coding_only=False,
               max_admm=500, outer=10),
    # C1 with J = 3 channels (Joint mode / TCSC; not a BASELINE config)
    "c1j3": dict(N=256, H=128, W=128, K=64, m=11, prec=32, beta=0.5, p=0.01, sigma=0.01, coding_only=True,
                 max_admm=50, outer=1, J=3),
    # C3-shaped slice for profiling only (not a BASELINE config)
    "c3s": dict(N=16, H=256, W=256, K=128, m=11, prec=32, beta=0.5, p=0.01, sigma=0.01, coding_only=True,
                max_admm=10, outer=1),
    "c4": dict(N=2048, H=64, W=64, K=32, m=7, prec=32, beta=0.5, p=0.005, sigma=0.05, coding_only=False,
               max_admm=500, outer=10),
}
SEED = 20250917


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_data(cfg, n0, n1):
    """Seeded synthetic signals of the config's shape. J > 1: channel j is the
    generator's output for seed SEED + j; the dictionary is the channel stack of
    the per-channel ground truths, jointly renormalised to unit filters."""
    from paper_1709_09479_b200 import dcsc
    J = cfg.get("J", 1)
    xs, ds = [], []
    for j in range(J):  # only this rank's images are generated (per-image streams)
        x, d_true = dcsc.synth_generate(n1 - n0, (cfg["H"], cfg["W"]), cfg["K"], cfg["m"], cfg["p"],
                                        cfg["sigma"], SEED + j, cfg["prec"] == 32, first=n0)
        xs.append(x)
        ds.append(d_true)
    if J == 1:
        return xs[0].copy(), ds[0]
    d = np.stack(ds, axis=1)
    d /= np.sqrt((d ** 2).sum(axis=(1, 2, 3), keepdims=True))
    return np.ascontiguousarray(np.stack(xs, axis=1)), d


def coding_bytes(cfg, n_img):
    """per ADMM iteration B = n*(4 K D s + J Dh 2s) + J K Dh 2s
    (J = 1 at the BASELINE configs)."""
    s = 4 if cfg["prec"] == 32 else 8
    D = cfg["H"] * cfg["W"]
    Dh = cfg["H"] * (cfg["W"] // 2 + 1)
    K = cfg["K"]
    J = cfg.get("J", 1)
    return n_img * (4 * K * D * s + J * Dh * 2 * s) + J * K * Dh * 2 * s


def traffic_from_profiles(name):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(name)
    except Exception:
        return None


# ---------------------------------------------------------------- reference arm
def ref_sample_coding(cfg, x, d, threads, admm_cap):
    from oracle import ref
    ref.set_threads(threads)
    n_img = min(len(x), max(threads, 1))
    c = ref.Cfg(beta=cfg["beta"], max_admm=admm_cap, normalize=0)
    t0 = time.perf_counter()
    if cfg.get("J", 1) > 1:
        iters, _ = ref.coding_batch_j(x[:n_img], d, c)
    else:
        iters, _ = ref.coding_batch(x[:n_img], d, c)
    dt = time.perf_counter() - t0
    # per-image ADMM iterations cost the same from a cold start; scale to N images x max_admm
    full = dt * (cfg["N"] * cfg["max_admm"]) / max(int(iters.sum()), 1)
    return full, dt, n_img, int(iters.sum())


def run_reference(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    x, d = make_data(cfg, 0, min(cfg["N"], max(threads, 1)))
    if not cfg["coding_only"]:
        return run_reference_full(args, cfg, x, threads)
    cap = 10
    for _ in range(args.warmup):
        ref_sample_coding(cfg, x, d, threads, 2)
    vals, dts = [], []
    for _ in range(args.steps):
        full, dt, n_img, it_sum = ref_sample_coding(cfg, x, d, threads, cap)
        vals.append(1.0 / full)
        dts.append(dt)
    value = float(np.median(vals))
    sample = (f"{n_img} of {cfg['N']} images x {cap} of {cfg['max_admm']} ADMM iters per step on {threads} threads "
              f"(OpenMP over images, pipeline.cpp:221), extrapolated linearly in images x iterations")
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / value, "higher_is_better": True,
        "scaling": "weak" if cfg["coding_only"] else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": config_block(cfg, args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return 0


def ref_sample_outer(cfg, x, threads, admm_cap):
    """One run_csc outer iteration of the reference on a subset of images with a
    capped ADMM budget, extrapolated to the full workload: coding scales with
    images x ADMM iterations (a cold start runs the whole budget), learning and
    the objective bookkeeping with images."""
    from oracle import ref
    ref.set_threads(threads)
    n_img = len(x)
    c = ref.Cfg(beta=cfg["beta"], max_admm=admm_cap, max_outer=1, normalize=0, seed=SEED, tol=1e-300)
    t0 = time.perf_counter()
    r = ref.run(x, cfg["K"], (cfg["m"], cfg["m"]), c, dump_dicts=False)
    wall = time.perf_counter() - t0
    rows = r["trace"]
    code_ms = rows[0]["elapsed_ms"]
    rest_ms = wall * 1e3 - code_ms
    full_ms = (code_ms * cfg["max_admm"] / admm_cap + rest_ms) * cfg["N"] / n_img
    return full_ms / 1e3, wall, n_img


def run_reference_full(args, cfg, x, threads):
    n_img = min(cfg["N"], max(2, min(threads, 8)))
    xs = x[:n_img]
    cap = 5
    for _ in range(args.warmup):
        ref_sample_outer(cfg, xs[:2], threads, 1)
    vals = []
    for _ in range(args.steps):
        full, wall, n = ref_sample_outer(cfg, xs, threads, cap)
        vals.append(1.0 / full)
    value = float(np.median(vals))
    sample = (f"one run_csc outer iteration on {n_img} of {cfg['N']} images, ADMM capped at {cap} of "
              f"{cfg['max_admm']}, {threads} threads; coding extrapolated x(images x iterations), learning and "
              f"objective x images (extrapolated estimate)")
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / value, "higher_is_better": True,
        "scaling": "weak" if cfg["coding_only"] else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": config_block(cfg, args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return 0


def config_block(cfg, args):
    name = args.config
    wl = (f"{name.upper()}: N={cfg['N']} images {cfg['H']}x{cfg['W']} FP{cfg['prec']}, K={cfg['K']} filters "
          f"{cfg['m']}x{cfg['m']}, beta={cfg['beta']}, rho=0.1, ")
    if cfg.get("J", 1) > 1:
        wl += f"J={cfg['J']} channels (Joint mode, TCSC), "
    if cfg["coding_only"]:
        wl += f"coding only, fixed ground-truth dictionary, {cfg['max_admm']} ADMM iters, cold start"
    else:
        wl += "coding+learning outer iteration of run_csc from init_variables"
    return {"workload": wl, "images": cfg["N"], "channels": cfg.get("J", 1), "filters": cfg["K"], "grid": [cfg["H"], cfg["W"]],
            "support": [cfg["m"], cfg["m"]], "precision": f"fp{cfg['prec']}", "parallelism": (f"dp{args.gpus}: {cfg['N']} images per GPU (weak)" if cfg["coding_only"]
                            else f"images sharded x{args.gpus} (strong)"),
            "l2": "inputs larger than L2 (ADMM state u = N*K*D*s)", "seed": SEED}


# ---------------------------------------------------------------- our arm
def run_ours(args, cfg):
    world, rank, local = dist_env()
    dist = None
    # DCSC_BENCH_DIST_BACKEND=gloo: host-side collectives (and the learning
    # all-reduce through the gloo host callback), so the multi-rank path can be
    # exercised with several ranks sharing one GPU; timings are then not scaling data.
    backend = os.environ.get("DCSC_BENCH_DIST_BACKEND", "nccl")
    dev = 0
    tdev = "cpu"
    if world > 1:
        import torch
        import torch.distributed as tdist
        dev = local % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(dev)
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", dev))
            tdev = "cuda"
        else:
            tdist.init_process_group("gloo")
        dist = tdist
    from paper_1709_09479_b200 import dcsc
    N = cfg["N"]
    # Coding-only configs shard the independent units (images) with no
    # collective: weak scaling, every rank codes its own N-image C1 workload
    # (rank r takes images [r N, (r+1) N) of one seeded N*world-image dataset),
    # so one step = `world` C1 outer iterations. Full configs (learning couples
    # the images through all-reduces) keep the N images and split them.
    weak = cfg["coding_only"]
    if weak:
        n0, n1 = rank * N, (rank + 1) * N
        x, d_true = make_data(cfg, n0, n1)
    else:
        n0, n1 = dcsc.shard_range(N, world, rank)
        x, d_true = make_data(cfg, n0, n1)
    nl = n1 - n0
    units = world if weak else 1  # C1-workload outer iterations per step, all ranks
    sc = dcsc.SolverConfig(beta=cfg["beta"], max_admm=cfg["max_admm"], normalize=0, seed=SEED, tol=1e-300)
    ctx = dcsc.Context(nl, (cfg["H"], cfg["W"]), cfg["K"], (cfg["m"], cfg["m"]), sc, cfg["prec"],
                       device=dev, channels=cfg.get("J", 1))
    if world > 1 and not cfg["coding_only"]:
        # learning sums its K x NB correlations and CG scalars over ranks (NCCL)
        import torch
        if backend == "nccl":
            uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if rank == 0:
                uid.copy_(torch.tensor(list(dcsc.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(uid, 0)
            ctx.set_comm_nccl(world, rank, bytes(uid.cpu().tolist()))
        else:
            ctx.set_comm_callback(world, rank, dcsc.gloo_allreduce_fn())
    ctx.set_signals(x)
    ctx.set_dictionary(d_true)

    def step():
        if cfg["coding_only"]:
            ctx.set_coding_state(None, None)
            return ctx.coding()
        return ctx.run(1)

    def barrier():
        if dist:
            dist.barrier()

    for _ in range(max(args.warmup, 0)):
        step()
    ctx.synchronize()
    barrier()
    ctx.set_profiling(2)  # per-launch events on the roofline kernel only (coding pass)
    l0 = ctx.kernel_launches()
    with ClockSampler(dev) as clk:
        ctx.event_mark(0)
        stats = None
        for _ in range(args.steps):
            stats = step()
        ctx.event_mark(1)
        ctx.synchronize()
    ms = ctx.event_elapsed(0, 1)
    launches = ctx.kernel_launches() - l0
    cod_ms, cod_n = ctx.kernel_time(0)
    # per-family breakdown from one extra, untimed step with every launch evented
    ctx.set_profiling(1)
    prof_step = step()
    ctx.synchronize()
    fam_names = ["coding_pass_admm", "lambda_update", "learning_contract", "learning_mask", "other"]
    fam_ms = {fam_names[f]: round(ctx.kernel_time(f)[0], 3) for f in range(5)}
    learn_ms, learn_n = ctx.kernel_time(2)  # z_hat streams (contract_c / contract_out) of that step
    if dist:
        import torch
        t = torch.tensor([ms], device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ctx.set_profiling(False)
    value = units * args.steps / (ms / 1000.0)

    # e2e through the C-ABI with host buffers: signals h2d + solve + stats d2h each step
    # each step timed on its own (host wall clock, synchronised); the median
    # step is reported, so one step disturbed by host noise does not set E
    e2e_steps = max(1, min(args.steps, 5))
    ctx.synchronize()
    barrier()
    step_s = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        ctx.set_signals(x)
        r = step()
        ctx.synchronize()
        step_s.append(time.perf_counter() - t0)
    e2e_s = statistics.median(step_s)
    if dist:
        import torch
        t = torch.tensor([e2e_s], device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = units / e2e_s
    s = 4 if cfg["prec"] == 32 else 8
    h2d = nl * cfg.get("J", 1) * cfg["H"] * cfg["W"] * s
    admm_max = max(st["admm_iters"] for st in stats) if cfg["coding_only"] else 0
    d2h = nl * (56 + 40) + nl * 4 * max(admm_max, 1)

    if rank != 0:
        return 0
    peak, peak_kind = load_peaks()
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak" if weak else "strong",
        "vs_baseline": None,
        "dtype": "f32" if cfg["prec"] == 32 else "f64", "data": "synthetic (seeded BASELINE.json generator)",
        "config": config_block(cfg, args),
        "e2e": {"value": e2e * 1.0, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "timing": f"median of {e2e_steps} host-timed steps (signals h2d + solve + stats d2h each)"},
        "gpu_launches": launches,
        "kernel_ms_per_step": fam_ms,
    }
    if cod_n:
        avg = cod_ms / cod_n
        # ADMM launches process every active image; cold start -> all images for max_admm iterations
        algo = coding_bytes(cfg, nl)
        achieved = algo / (avg / 1000.0) / 1e9
        out["roofline"] = {"bound": "hbm", "kernel": "coding_pass<ADMM>", "achieved": achieved, "peak": peak,
                           "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                           "traffic": traffic_from_profiles(args.config), "algorithmic_bytes_per_launch": algo,
                           "avg_launch_ms": avg, "launches": cod_n,
                           "share_of_step": cod_ms / ms}
    if learn_n and not cfg["coding_only"]:
        # learning's z_hat streams over the profiled outer iteration: each CG
        # apply (cg_iters + one warm-start residual apply per mu iteration) is one
        # contract_c + one contract_out, each d_recover one contract_c; launches
        # issued past the device-side CG stop exit at once and are not counted
        rows = [r for r in prof_step[0] if r["phase"] == 1] if isinstance(prof_step, tuple) else []
        cg_it = sum(r["cg_iters"] for r in rows)
        mu_it = sum(r["mu_iters"] for r in rows)
        streams = 2 * (cg_it + mu_it) + mu_it
        if streams > 0:
            sc = 8 if cfg["prec"] == 32 else 16
            nbins = cfg["H"] * (cfg["W"] // 2 + 1)
            per = (nl * cfg["K"] + 3 * nl + cfg["K"]) * nbins * sc  # z_hat + v/out + p_hat per launch
            ach = per * streams / (learn_ms / 1000.0) / 1e9
            out["roofline_learning"] = {
                "bound": "hbm", "kernel": "contract_c / contract_out (z_hat streams)", "achieved": ach,
                "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": ach / peak,
                "algorithmic_bytes_per_launch": per, "launches_counted": streams, "cg_iters": cg_it,
                "mu_iters": mu_it, "kernel_ms": learn_ms,
                "note": "one extra, untimed outer iteration with every launch evented"}
    out["clocks"] = clk.summary()
    if world == 1 and not args.no_cpu_baseline and cfg["coding_only"]:
        try:
            threads = os.cpu_count() or 1
            xs, d = make_data(cfg, 0, min(cfg["N"], threads))
            full, dt, n_img, it_sum = ref_sample_coding(cfg, xs, d, threads, 10)
            out["cpu_baseline"] = {
                "value": 1.0 / full, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"{n_img} images x 10 ADMM iters ({dt:.1f}s wall), extrapolated to {cfg['N']} x "
                          f"{cfg['max_admm']}; FFT via oracle/fftw_shim.c (FFTW absent)"}
        except Exception as e:  # the checker must not take the bench down
            out["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                                   "sample": f"unavailable: {e}"}
    elif world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            xs, _ = make_data(cfg, 0, min(cfg["N"], 4))
            full, wall, n = ref_sample_outer(cfg, xs, threads, 3)
            out["cpu_baseline"] = {
                "value": 1.0 / full, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"one run_csc outer iteration on {n} images, ADMM capped at 3 ({wall:.1f}s wall), "
                          f"extrapolated to {cfg['N']} images x {cfg['max_admm']} ADMM iters (estimate)"}
        except Exception as e:
            out["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                                   "sample": f"unavailable: {e}"}
    print(json.dumps(out))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
