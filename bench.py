#!/usr/bin/env python3
"""Benchmark of the B200 dual-domain CSC hot path (BASELINE.json metric).

Default workload (N=1): BASELINE.json configs[3] (C3), the largest config and
the one the metric's "outer iters/s (coding+learning)" is quoted on at 1-8
GPUs: N=512 images 256x256 FP32, K=128 filters 11x11, beta=0.5, rho=0.1, 10
outer iterations. One step = the NEXT outer iteration of one continuous
run_csc run (pipeline.cpp:216-299: coding of every image, the objective /
acceptance bookkeeping, one solve_learning), through the run_begin / run_step
entry points; the run restarts from init_variables every 10 outer iterations
(the config's length), so W warm-up steps then K timed steps cover outer
iterations W+1 .. W+K of that cycle. --config c0/c2/c4 run the other full
configs the same way; c1 (coding only, 50 ADMM iterations, cold start),
c1j3 (C1 with J=3) and c3s (a 16-image C3 coding slice) time one coding pass.

value  = outer iterations/s with the inputs resident in HBM (device events on
         the library stream, max over ranks).
e2e    = the same metric through the public API with host buffers: each step
         uploads the signals from host memory (set_signals), runs the outer
         iteration and returns what run_csc returns per outer iteration (the
         two trace rows and the dictionary). Maps and the ADMM / CG state stay
         on the device by design.
Multi-GPU: `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks (one per GPU, NCCL). Full configs split
their N images over the ranks (strong scaling; learning all-reduces its K x M
crops and CG scalars over NCCL); coding-only configs give every rank its own
C1 workload (weak scaling).

--impl reference times the reference's own CPU implementation (oracle/_ref:
the unmodified reference solver TUs) on the box's host cores, from measured
unit costs on a bounded sample (see ref_unit_costs), composed with the same
outer iterations' work counts.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
    # name: N, H, W, K, m, precision, beta, p, sigma, coding_only, max_admm, outer (run length)
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
    # C3-shaped coding slice for profiling only (not a BASELINE config); 16 images are below the
    # tensor-core pass's default batch threshold, so it is forced (DCSC_TC=1) to profile C3's kernel
    "c3s": dict(N=16, H=256, W=256, K=128, m=11, prec=32, beta=0.5, p=0.01, sigma=0.01, coding_only=True,
                max_admm=10, outer=1, env={"DCSC_TC": "1"}),
    # a 128-image C3 coding slice for A/B timing of the coding pass under load (~14 work items per SM)
    "c3m": dict(N=128, H=256, W=256, K=128, m=11, prec=32, beta=0.5, p=0.01, sigma=0.01, coding_only=True,
                max_admm=20, outer=1),
    "c4": dict(N=2048, H=64, W=64, K=32, m=7, prec=32, beta=0.5, p=0.005, sigma=0.05, coding_only=False,
               max_admm=500, outer=10),
}
SEED = 20250917
DEFAULT_CONFIG = "c3"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_tensor_peak():
    """Dense f16/bf16 tensor peak (TFLOP/s) from MEASURED_PEAKS.json: the sustained figure (the coding
    pass is timed inside a long step, back to back for seconds), with the burst figure beside it; else the
    recipe's nominal. Returns (peak, kind, burst or None)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        burst = float(p["bf16_tflops"])
        if p.get("bf16_tflops_sustained"):
            return float(p["bf16_tflops_sustained"]), "measured (sustained)", burst
        return burst, "measured (burst)", burst
    except Exception:
        return 2250.0, "fallback", None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,enforced.power.limit")

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
        sm, mx, reasons, pw, plim = [], None, set(), [], None
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
            try:  # board power during the timed region against the enforced limit (explains sw_power_cap)
                pw.append(float(parts[2]))
                plim = float(parts[7]) if len(parts) > 7 else plim
            except ValueError:
                pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}
        if pw:
            out["power_w"] = statistics.median(pw)
            out["power_limit_w"] = plim
        return out


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def spawn_ranks(args) -> int | None:
    """`--gpus N` outside torchrun: re-launch this script under
    torch.distributed.run with N ranks on 127.0.0.1 (one process per GPU)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def make_data(cfg, n0, n1, gen=None):
    """Seeded synthetic signals of the config's shape (images [n0, n1)). `gen` is
    the generator function: dcsc.synth_generate on our arm, ref.synth_generate (the
    same source compiled into the oracle library) on the reference arm. J > 1:
    channel j is the generator's output for seed SEED + j; the dictionary is the
    channel stack of the per-channel ground truths, jointly renormalised."""
    if gen is None:
        from paper_1709_09479_b200 import dcsc
        gen = dcsc.synth_generate
    J = cfg.get("J", 1)
    xs, ds = [], []
    for j in range(J):
        x, d_true = gen(n1 - n0, (cfg["H"], cfg["W"]), cfg["K"], cfg["m"], cfg["p"], cfg["sigma"], SEED + j,
                        cfg["prec"] == 32, first=n0)
        xs.append(x)
        ds.append(d_true)
    if J == 1:
        return xs[0].copy(), ds[0]
    d = np.stack(ds, axis=1)
    d /= np.sqrt((d ** 2).sum(axis=(1, 2, 3), keepdims=True))
    return np.ascontiguousarray(np.stack(xs, axis=1)), d


def sizes(cfg):
    s = 4 if cfg["prec"] == 32 else 8
    D = cfg["H"] * cfg["W"]
    Dh = cfg["H"] * (cfg["W"] // 2 + 1)
    return s, D, Dh


def coding_bytes(cfg, n_img):
    """per ADMM iteration B = n*(4 K D s + J Dh 2s) + J K Dh 2s."""
    s, D, Dh = sizes(cfg)
    K, J = cfg["K"], cfg.get("J", 1)
    return n_img * (4 * K * D * s + J * Dh * 2 * s) + J * K * Dh * 2 * s


def outer_bytes(cfg, n_img, admm_total, admm_rounds, cg_iters, mu_iters):
    """SURVEY.md §8(d) compulsory bytes of one outer iteration:
    B_code + B_learn + B_obj (dense-state formula, a minimum)."""
    s, D, Dh = sizes(cfg)
    K, N = cfg["K"], n_img
    b_code = admm_total * (4 * K * D * s + Dh * 2 * s) + admm_rounds * K * Dh * 2 * s
    b_learn = (N * K * (D * s + Dh * 2 * s) + (cg_iters + mu_iters) * (2 * N * K * Dh * 2 * s + 6 * N * Dh * 2 * s
               + 2 * K * Dh * 2 * s) + mu_iters * N * K * Dh * 2 * s)
    b_obj = N * K * D * s
    return b_code, b_learn, b_obj


def traffic_from_profiles(name):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(name)
    except Exception:
        return None


def counts_file(name):
    return os.path.join(ROOT, "profiles", f"counts_{name}.json")


def timed_outer_indices(cfg, warmup, steps):
    """Outer-iteration indices (1-based, within the restart cycle) of the timed steps."""
    L = cfg["outer"]
    return [((warmup + i) % L) + 1 for i in range(steps)]


# ---------------------------------------------------------------- reference CPU costs
def ref_unit_costs(cfg, threads):
    """Measured unit costs of the reference's own code (oracle/_ref, the
    unmodified solver TUs) on this host, on a bounded sample:
      coding:    wall per image-ADMM-iteration and per-solve set-up, from two
                 OpenMP batches over `threads` images (ADMM capped at 1 and 3;
                 coding is image-parallel as pipeline.cpp:221);
      objective: one evaluate_objective (objective.cpp:59-81; serial over
                 images in run_csc, pipeline.cpp:232-282) on one image;
      learning:  LearningOperator build (N*K FFTs) and apply at n_s and 2 n_s
                 images (linear fit in N: apply = 2N+2K FFTs + 2NKD MACs)."""
    from oracle import ref
    ref.set_threads(threads)
    n_s = max(2, min(threads, cfg["N"]))
    x, d = make_data(cfg, 0, n_s, ref.synth_generate)
    if cfg.get("J", 1) > 1:
        raise RuntimeError("reference unit costs are for J = 1 configs")
    ref.coding_batch(x[: min(2, n_s)], d, ref.Cfg(beta=cfg["beta"], max_admm=1, normalize=0))  # untimed: plans, threads
    tc = {}
    for cap in (1, 3):
        c = ref.Cfg(beta=cfg["beta"], max_admm=cap, normalize=0)
        t0 = time.perf_counter()
        iters, _ = ref.coding_batch(x, d, c)
        tc[cap] = (time.perf_counter() - t0, int(iters.sum()))
    per_iter = max((tc[3][0] - tc[1][0]) / max(tc[3][1] - tc[1][1], 1), 1e-9)
    per_solve = max(tc[1][0] / n_s - per_iter, 0.0)
    out = {"n_sample": n_s, "coding_iter_s": per_iter, "coding_setup_s": per_solve,
           "coding_sample_s": tc[1][0] + tc[3][0]}
    rng = np.random.default_rng(1)
    z = (rng.random((1, cfg["K"], cfg["H"], cfg["W"])) < cfg["p"]) * rng.laplace(size=(1, cfg["K"], cfg["H"], cfg["W"]))
    t0 = time.perf_counter()
    ref.set_threads(1)
    ref.objective(x[0], d, z[0], cfg["beta"])
    out["objective_s"] = time.perf_counter() - t0
    ref.set_threads(threads)
    if not cfg["coding_only"]:
        lt = {}
        for n in (n_s, 4 * n_s):
            maps = (rng.random((n, cfg["K"], cfg["H"], cfg["W"])) < cfg["p"]) * 1.0
            b, a = ref.time_learning(maps, (cfg["m"], cfg["m"]), 3)
            lt[n] = (b / 1e3, a / 1e3)
        # linear fit in N through the two sizes (the per-image slope is floored at
        # the large sample's mean share, so timer noise cannot zero it)
        slope_a = max((lt[4 * n_s][1] - lt[n_s][1]) / (3 * n_s), 0.25 * lt[4 * n_s][1] / (4 * n_s))
        icpt_a = max(lt[n_s][1] - slope_a * n_s, 0.0)
        slope_b = max((lt[4 * n_s][0] - lt[n_s][0]) / (3 * n_s), lt[4 * n_s][0] / (4 * n_s))
        out.update({"apply_s_per_image": slope_a, "apply_s_fixed": icpt_a, "build_s_per_image": slope_b})
    return out


def ref_outer_seconds(cfg, uc, n_img, counts):
    """Reference wall seconds of one outer iteration on this host with the given
    work counts: coding (admm_total image-iterations + per-image set-up, packed
    over the OpenMP threads as measured), 3 objective passes per image
    (pipeline.cpp:234, 269-270 learning_data_term, 282), learning (operator
    build + (cg_iters + mu_iters) applies + mu_iters d_recover at ~half an apply).
    Coding-only configs (C1) time solve_coding of every image and nothing else."""
    code = counts["admm_total"] * uc["coding_iter_s"] + n_img * uc["coding_setup_s"]
    obj = 0.0 if cfg["coding_only"] else 3 * n_img * uc["objective_s"]
    learn = 0.0
    if not cfg["coding_only"]:
        apply_s = uc["apply_s_fixed"] + uc["apply_s_per_image"] * n_img
        learn = (uc["build_s_per_image"] * n_img + (counts["cg_iters"] + counts["mu_iters"]) * apply_s
                 + 0.5 * counts["mu_iters"] * apply_s)
    return code + obj + learn, {"coding_s": code, "objective_s": obj, "learning_s": learn}


def load_counts(name, cfg, idx):
    """Per-outer work counts (admm_total, cg_iters, mu_iters) of this config's run
    at the given outer indices, from profiles/counts_<config>.json (written by
    `bench.py --dump-counts` on the GPU; the FP64 reference takes the same ADMM,
    CG and mu iteration counts, tests/test_golden_gpu.py). Fallback: the caps."""
    try:
        with open(counts_file(name)) as f:
            per = {int(k): v for k, v in json.load(f)["per_outer"].items()}
        return [per[i] for i in idx], "profiles/" + os.path.basename(counts_file(name))
    except Exception:
        c = {"admm_total": cfg["N"] * cfg["max_admm"], "cg_iters": 300, "mu_iters": 1}
        return [c for _ in idx], "budget caps (counts file missing)"


def run_reference(args, cfg):
    """--impl reference: the reference's own CPU implementation (oracle/_ref) on
    this host's cores. Each step re-measures the unit costs on a bounded sample
    (ref_unit_costs) and composes one outer iteration of the timed workload."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    if cfg.get("J", 1) > 1:  # Joint mode: image-proportional sample
        return run_reference_sample_j(args, cfg, threads)
    idx = timed_outer_indices(cfg, args.warmup, args.steps) if not cfg["coding_only"] else [1] * args.steps
    counts, src = (load_counts(args.config, cfg, idx) if not cfg["coding_only"]
                   else ([{"admm_total": cfg["N"] * cfg["max_admm"]}] * args.steps, "cold start: N x max_admm"))
    for _ in range(args.warmup):
        ref_unit_costs(dict(cfg, N=min(cfg["N"], 4)), threads)
    secs, samples, parts = [], [], None
    for i in range(args.steps):
        t0 = time.perf_counter()
        uc = ref_unit_costs(cfg, threads)
        samples.append(time.perf_counter() - t0)
        s, parts = ref_outer_seconds(cfg, uc, cfg["N"], counts[i])
        secs.append(s)
    value = len(secs) / sum(secs)
    assert_no_product_library()
    sample = (f"unit costs of the reference code measured per step on this host ({threads} threads, "
              f"{uc['n_sample']}-image samples: coding capped at 1 and 3 ADMM iters, one objective, learning "
              f"operator at {uc['n_sample']} and {2 * uc['n_sample']} images; {statistics.median(samples):.1f}s of CPU "
              f"work per step), composed with the timed outer iterations' work counts ({src}); "
              f"extrapolated estimate, FFT = oracle/fftw_shim.c (FFTW absent)")
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / value, "higher_is_better": True,
        "scaling": "weak" if cfg["coding_only"] else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE.json generator)", "config": config_block(cfg, args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample,
                         "extrapolated": True, "sample_seconds_per_step": round(statistics.median(samples), 2),
                         "seconds_per_outer_breakdown": {k: round(v, 2) for k, v in parts.items()},
                         "unit_costs": {k: (round(v, 6) if isinstance(v, float) else v) for k, v in uc.items()}},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "timed_outer_iters": idx if not cfg["coding_only"] else None,
    }
    print(json.dumps(out))
    return 0


def assert_no_product_library():
    """The reference arm runs only the reference (oracle/_ref): fail loudly if the
    CUDA product library got mapped into this process."""
    try:
        with open("/proc/self/maps") as f:
            if "libdcsc_cuda" in f.read():
                raise RuntimeError("reference arm mapped libdcsc_cuda.so")
    except FileNotFoundError:
        pass


def run_reference_sample_j(args, cfg, threads):
    from oracle import ref
    ref.set_threads(threads)
    x, d = make_data(cfg, 0, min(cfg["N"], threads), ref.synth_generate)
    cap = 10
    vals = []
    for i in range(args.warmup + args.steps):
        c = ref.Cfg(beta=cfg["beta"], max_admm=cap if i >= args.warmup else 2, normalize=0)
        t0 = time.perf_counter()
        iters, _ = ref.coding_batch_j(x, d, c)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            vals.append(1.0 / (dt * cfg["N"] * cfg["max_admm"] / max(int(iters.sum()), 1)))
    value = float(np.median(vals))
    assert_no_product_library()
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 / value, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE.json generator)",
        "config": config_block(cfg, args, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{len(x)} images x {cap} ADMM iters per step, extrapolated to N x max_admm"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return 0


def config_block(cfg, args, world):
    name = args.config
    wl = (f"{name.upper()}: N={cfg['N']} images {cfg['H']}x{cfg['W']} FP{cfg['prec']}, K={cfg['K']} filters "
          f"{cfg['m']}x{cfg['m']}, beta={cfg['beta']}, rho=0.1, ")
    if cfg.get("J", 1) > 1:
        wl += f"J={cfg['J']} channels (Joint mode, TCSC), "
    if cfg["coding_only"]:
        wl += f"coding only, fixed ground-truth dictionary, {cfg['max_admm']} ADMM iters, cold start"
    else:
        wl += (f"one coding+learning outer iteration of a continuous run_csc run per step (restarted from "
               f"init_variables every {cfg['outer']} outer iterations), max_admm={cfg['max_admm']}")
    return {"workload": wl, "images": cfg["N"], "channels": cfg.get("J", 1), "filters": cfg["K"],
            "grid": [cfg["H"], cfg["W"]], "support": [cfg["m"], cfg["m"]], "precision": f"fp{cfg['prec']}",
            "parallelism": (f"{cfg['N']} images per GPU x {world} GPUs (weak)" if cfg["coding_only"]
                            else f"{cfg['N']} images sharded over {world} GPU(s) (strong), learning "
                                 f"{getattr(args, 'learning_layout', 'image')}-sharded"),
            "l2": "inputs larger than L2 (ADMM state u = N*K*D*s)", "seed": SEED}


# ---------------------------------------------------------------- our arm
def setup_dist(world, local):
    backend = os.environ.get("DCSC_BENCH_DIST_BACKEND", "nccl")
    dev, dist, tdev = 0, None, "cpu"
    if world > 1:
        import torch
        import torch.distributed as tdist
        ndev = torch.cuda.device_count()
        if backend == "nccl" and ndev < world:
            raise RuntimeError(f"{world} NCCL ranks need {world} GPUs, {ndev} visible "
                               "(DCSC_BENCH_DIST_BACKEND=gloo shares one GPU for functional runs)")
        dev = local % max(ndev, 1)
        torch.cuda.set_device(dev)
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", dev))
            tdev = "cuda"
        else:
            tdist.init_process_group("gloo")
        dist = tdist
    return dev, dist, tdev, backend


def run_ours(args, cfg):
    world, rank, local = dist_env()
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (nranks) on stderr
    dev, dist, tdev, backend = setup_dist(world, local)
    from paper_1709_09479_b200 import dcsc

    def max_over_ranks(v):
        if not dist:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64, device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v):
        if not dist:
            return v
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64, device=tdev)
        dist.all_reduce(t)
        return float(t.item())

    def barrier():
        if dist:
            dist.barrier()

    N = cfg["N"]
    weak = cfg["coding_only"]
    if weak:  # every rank codes its own N-image workload: rank r takes images [r N, (r+1) N)
        n0, n1 = rank * N, (rank + 1) * N
    else:
        n0, n1 = dcsc.shard_range(N, world, rank)
    x, d_true = make_data(cfg, n0, n1, dcsc.synth_generate)
    nl = n1 - n0
    sc = dcsc.SolverConfig(beta=cfg["beta"], max_admm=cfg["max_admm"], normalize=0, seed=SEED, tol=1e-300)
    ctx = dcsc.Context(nl, (cfg["H"], cfg["W"]), cfg["K"], (cfg["m"], cfg["m"]), sc, cfg["prec"],
                       device=dev, channels=cfg.get("J", 1))
    coding_path = ctx.coding_path()
    nccl_ranks = None
    if world > 1 and not weak:
        import torch
        if backend == "nccl":
            uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if rank == 0:
                uid.copy_(torch.tensor(list(dcsc.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(uid, 0)
            ctx.set_comm_nccl(world, rank, bytes(uid.cpu().tolist()))
            nccl_ranks = world
        else:
            ctx.set_comm_callback(world, rank, dcsc.gloo_allreduce_fn())
        ctx.set_learning_layout(args.learning_layout)
    ctx.set_signals(x)
    ctx.set_dictionary(d_true)

    state = {"outer": 0}

    def full_step():
        if state["outer"] >= cfg["outer"]:
            ctx.run_begin()
            state["outer"] = 0
        rows, _ = ctx.run_step()
        state["outer"] += 1
        return rows

    def coding_step():
        ctx.set_coding_state(None, None)
        return ctx.coding()

    step = coding_step if weak else full_step
    if not weak:
        ctx.run_begin()

    # ---- warm-up, then K device-timed steps (inputs resident)
    for _ in range(max(args.warmup, 0)):
        step()
    ctx.synchronize()
    barrier()
    # per-launch events on the dominant kernel family (coding pass) and, for
    # full configs, the learning z_hat streams (contract_c / contract_out)
    ctx.set_profiling(2 if weak else 3)
    l0 = ctx.kernel_launches()
    rows_timed, stats = [], None
    with ClockSampler(dev) as clk:
        ctx.event_mark(0)
        for _ in range(args.steps):
            r = step()
            if weak:
                stats = r
            else:
                rows_timed.extend(r)
        ctx.event_mark(1)
        ctx.synchronize()
    ms_local = ctx.event_elapsed(0, 1)
    launches = ctx.kernel_launches() - l0
    cod_ms, cod_n = ctx.kernel_time(0)
    learn_ms, learn_n = ctx.kernel_time(2)
    ctx.set_profiling(0)
    ms = max_over_ranks(ms_local)
    units = world if weak else 1
    value = units * args.steps / (ms / 1000.0)
    timed_idx = timed_outer_indices(cfg, args.warmup, args.steps) if not weak else None

    # ---- e2e through the public API with host buffers, the next steps of the run
    e2e_steps = max(1, min(args.steps, 3))
    barrier()
    step_s, d2h = [], 0
    rows_e2e = []
    for _ in range(e2e_steps):
        ctx.synchronize()
        t0 = time.perf_counter()
        ctx.set_signals(x)                       # h2d of this step's inputs (pinned staging)
        r = step()
        if weak:
            out_bytes = sum(8 * 9 for _ in r)    # per-image coding stats
        else:
            dct = ctx.get_dictionary()           # what run_csc returns per outer: trace rows + dictionary
            out_bytes = dct.nbytes + 2 * 88
            rows_e2e.extend(r)
        ctx.synchronize()
        step_s.append(time.perf_counter() - t0)
        d2h = out_bytes
    e2e_s = max_over_ranks(sum(step_s) / len(step_s))
    e2e = units / e2e_s
    s_bytes = 4 if cfg["prec"] == 32 else 8
    h2d = nl * cfg.get("J", 1) * cfg["H"] * cfg["W"] * s_bytes

    # per-family breakdown (device ms) and counts over the timed region
    admm_total = sum(r["admm_iters"] for r in rows_timed if r["phase"] == 0)
    cg_it = sum(r["cg_iters"] for r in rows_timed if r["phase"] == 1)
    mu_it = sum(r["mu_iters"] for r in rows_timed if r["phase"] == 1)
    cod_ms_all = max_over_ranks(cod_ms)
    if rank != 0:
        ctx.close()
        return 0
    peak, peak_kind = load_peaks()
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak" if weak else "strong",
        "vs_baseline": None,
        "dtype": "f32" if cfg["prec"] == 32 else "f64", "data": "synthetic (seeded BASELINE.json generator)",
        "config": config_block(cfg, args, world),
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "timing": (f"mean of {e2e_steps} host-timed steps: signals h2d + the step + its outputs d2h "
                           + ("(per-image stats)" if weak else "(trace rows + dictionary; maps / state stay "
                                                             "device-resident by design)")),
                "outer_iters": ([r["outer_iter"] for r in rows_e2e if r["phase"] == 0] if not weak else None)},
        "gpu_launches": launches,
        "coding_path": coding_path,
    }
    if not weak:
        out["timed_outer_iters"] = timed_idx
        out["work_counts"] = {"admm_iters": admm_total, "cg_iters": cg_it, "mu_iters": mu_it,
                              "per_outer": [{"outer": rows_timed[2 * i]["outer_iter"],
                                             "admm_total": rows_timed[2 * i]["admm_iters"],
                                             "cg_iters": rows_timed[2 * i + 1]["cg_iters"],
                                             "mu_iters": rows_timed[2 * i + 1]["mu_iters"]}
                                            for i in range(len(rows_timed) // 2)]}
    if cod_n:
        avg = cod_ms / cod_n
        if weak:
            # cold start: every image runs every ADMM launch (max_admm iterations)
            algo_total = coding_bytes(cfg, nl) * cod_n
        else:
            # admm_total image-iterations + one d_hat read per launch
            s, D, Dh = sizes(cfg)
            algo_total = (admm_total / world * (4 * cfg["K"] * D * s + Dh * 2 * s)
                          + cod_n * cfg["K"] * Dh * 2 * s)
        achieved = algo_total / (cod_ms / 1000.0) / 1e9
        if coding_path == "tensor":
            # tcgen05 spatial pass: the u state (read + write) is the kernel's
            # minimum HBM traffic (2 K D s per image-iteration, plus the f16
            # lambda band and the col2im band partials, 13/8 of a plane each);
            # SURVEY.md 8(d)'s formula charges theta and z separately (twice
            # the bytes of u) and is kept as formula_bytes_per_launch
            s_, D_, _ = sizes(cfg)
            # Large batches run as two half-batches on two streams whose launches
            # overlap (one half's per-iteration neighbours beside the other half's
            # pass), so per-launch event times double-count; the rate is taken over
            # the coding phase's device time instead (the passes plus their
            # neighbours: a lower bound on the pass's own rate).
            if weak:  # cold start: every image runs every ADMM iteration
                img_it = nl * cfg["max_admm"] * args.steps
                phase_ms = ms
            else:
                img_it = admm_total / world
                phase_ms = sum(r["elapsed_ms"] for r in rows_timed if r["phase"] == 0)
            kern_bytes = img_it * (2 * cfg["K"] * D_ * s_ + 2 * (26 / 16) * D_ * 4)
            ach_b = kern_bytes / (phase_ms / 1000.0) / 1e9
            kf = (32 if cfg["K"] <= 32 else 64) if cfg["W"] == 64 else (64 if cfg["K"] <= 64 else 128)
            tp = 64 if cfg["m"] * cfg["m"] <= 64 else 128
            # 2 GEMMs x 3 f16 products x 2 flops x TP taps x KF filter slots per pixel
            flops = img_it * D_ * 12 * tp * kf
            ach_f = flops / (phase_ms / 1000.0) / 1e12
            tpeak, tpk, tburst = load_tensor_peak()
            out["roofline"] = {"bound": "hbm", "kernel": "coding_pass_tc (tcgen05 spatial ADMM iteration)",
                               "achieved": ach_b, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                               "frac": ach_b / peak, "traffic": traffic_from_profiles(args.config + "_tc"),
                               "algorithmic_bytes": kern_bytes, "coding_phase_ms": phase_ms,
                               "algorithmic_bytes_per_launch": kern_bytes / cod_n,
                               "formula_bytes_per_launch": algo_total / cod_n,
                               "avg_launch_ms": avg, "launches": cod_n, "share_of_step": min(1.0, phase_ms / ms),
                               "timing": "bytes / coding-phase device time (passes + per-iteration neighbours)"}
            out["roofline_tensor"] = {"bound": "tensor", "kernel": "coding_pass_tc (f16 x3 split GEMMs)",
                                      "achieved": ach_f, "peak": tpeak, "peak_kind": tpk, "unit": "TFLOP/s",
                                      "frac": ach_f / tpeak, "flops": flops, "peak_burst": tburst,
                                      "frac_of_burst": (ach_f / tburst if tburst else None)}
        else:
            out["roofline"] = {"bound": "hbm", "kernel": "coding_pass<ADMM> (coding_pass_cl at 256x256)",
                               "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                               "frac": achieved / peak, "traffic": traffic_from_profiles(args.config),
                               "algorithmic_bytes_per_launch": algo_total / cod_n, "avg_launch_ms": avg,
                               "launches": cod_n, "share_of_step": cod_ms_all / ms}
    if learn_n and not weak:
        # z_hat streams: each CG apply (cg_iters + one warm-start residual apply per
        # mu iteration) is one contract_c + one contract_out, each d_recover one
        # contract_c; launches issued past the device-side CG stop exit at once
        streams = 2 * (cg_it + mu_it) + mu_it
        s, D, Dh = sizes(cfg)
        sc8 = 2 * s
        per = (nl * cfg["K"] + 3 * nl + cfg["K"]) * Dh * sc8
        ach = per * streams / (learn_ms / 1000.0) / 1e9
        out["roofline_learning"] = {
            "bound": "hbm", "kernel": "contract_c / contract_out (z_hat streams)", "achieved": ach, "peak": peak,
            "peak_kind": peak_kind, "unit": "GB/s", "frac": ach / peak, "algorithmic_bytes_per_launch": per,
            "launches_counted": streams, "kernel_ms": learn_ms, "share_of_step": learn_ms / ms}
        b_code, b_learn, b_obj = (0, 0, 0)
        for i in range(len(rows_timed) // 2):
            rc, rl = rows_timed[2 * i], rows_timed[2 * i + 1]
            bc, bl, bo = outer_bytes(cfg, nl, rc["admm_iters"] / world, cfg["max_admm"], rl["cg_iters"],
                                     rl["mu_iters"])
            b_code, b_learn, b_obj = b_code + bc, b_learn + bl, b_obj + bo
        tot = b_code + b_learn + b_obj
        out["roofline_step"] = {
            "bound": "hbm", "kernel": "whole outer iteration (SURVEY.md §8(d) B_code + B_learn + B_obj)",
            "achieved": tot / (ms_local / 1000.0) / 1e9, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
            "frac": tot / (ms_local / 1000.0) / 1e9 / peak,
            "bytes": {"code": b_code, "learn": b_learn, "obj": b_obj}}
    if nccl_ranks:
        out["nccl_ranks"] = nccl_ranks
    out["clocks"] = clk.summary()
    if world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            t0 = time.perf_counter()
            if cfg.get("J", 1) > 1:
                raise RuntimeError("Joint-mode configs: see --impl reference")
            uc = ref_unit_costs(cfg, threads)
            wall = time.perf_counter() - t0
            if weak:
                counts = [{"admm_total": cfg["N"] * cfg["max_admm"]}]
            else:
                counts = out["work_counts"]["per_outer"]
            secs = [ref_outer_seconds(cfg, uc, cfg["N"], c)[0] for c in counts]
            out["cpu_baseline"] = {
                "value": len(secs) / sum(secs), "unit": UNIT, "cores": threads, "kind": "reference",
                "extrapolated": True, "sample_seconds": round(wall, 2),
                "sample": (f"reference unit costs measured on {uc['n_sample']}-image samples ({wall:.1f}s wall on "
                           f"{threads} threads: coding capped at 1 and 3 ADMM iters, one objective"
                           + (", learning operator build/apply at two sizes" if not weak else "")
                           + "), composed with the timed steps' own work counts; extrapolated estimate")}
        except Exception as e:  # the checker must not take the bench down
            out["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                                   "sample": f"unavailable: {e}"}
    print(json.dumps(out), flush=True)
    ctx.close()
    return 0


def dump_counts(args, cfg):
    """Run one whole restart cycle (cfg['outer'] outer iterations) on one GPU and
    write the per-outer work counts to profiles/counts_<config>.json (the
    reference arm composes its unit costs with these)."""
    from paper_1709_09479_b200 import dcsc
    x, d_true = make_data(cfg, 0, cfg["N"], dcsc.synth_generate)
    sc = dcsc.SolverConfig(beta=cfg["beta"], max_admm=cfg["max_admm"], normalize=0, seed=SEED, tol=1e-300)
    per = {}
    with dcsc.Context(cfg["N"], (cfg["H"], cfg["W"]), cfg["K"], (cfg["m"], cfg["m"]), sc, cfg["prec"]) as ctx:
        ctx.set_signals(x)
        ctx.run_begin()
        for o in range(1, cfg["outer"] + 1):
            t0 = time.perf_counter()
            rows, _ = ctx.run_step()
            per[o] = {"admm_total": rows[0]["admm_iters"], "cg_iters": rows[1]["cg_iters"],
                      "mu_iters": rows[1]["mu_iters"], "l0": rows[0]["l0"], "total": rows[1]["total"],
                      "coding_ms": rows[0]["elapsed_ms"], "learning_ms": rows[1]["elapsed_ms"],
                      "wall_s": time.perf_counter() - t0}
            print(json.dumps({"outer": o, **per[o]}), flush=True)
    with open(counts_file(args.config), "w") as f:
        json.dump({"config": args.config, "per_outer": per}, f, indent=1)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dump-counts", action="store_true")
    ap.add_argument("--learning-layout", default="image", choices=["image", "freq"],
                    help="multi-GPU learning: image-sharded (crop all-reduce) or frequency-sharded "
                         "(z_hat all-to-all per outer iteration)")
    args = ap.parse_args()
    rc = spawn_ranks(args)
    if rc is not None:
        return rc
    cfg = CONFIGS[args.config]
    for k, v in cfg.get("env", {}).items():
        os.environ.setdefault(k, v)
    if args.dump_counts:
        return dump_counts(args, cfg)
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
