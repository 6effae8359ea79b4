#!/usr/bin/env python
"""Kron-STAP frame throughput on B200 (pixels/s), per the graft bench contract.

Workload (BASELINE.json configs[1]): one Gotcha-scale frame
per GPU per step -- 3 channels x 2001 pulses x 2001 range bins, 2001 Doppler
bins x 16 spatial candidates, ranks (1, 3), tol 1e-4 -- run end to end
(sample covariance -> LR-Kron estimate -> filter bases -> detection map).
A pixel is one (range bin, Doppler) entry of the detection map.
N > 1 (torchrun): frame sharding (configs[2]); every rank processes its own
frame each step, no data-path collective; timing is the max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
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

CONFIGS = {
    # name: (p, q, n_bins, D, G, ra, rb, K passes)
    "gotcha": (3, 2001, 2001, 2001, 16, 1, 3, 1),
    "cfg1": (3, 256, 256, 256, 16, 1, 3, 1),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="gotcha",
                    choices=sorted(CONFIGS) + ["lmode", "multipass", "sweep"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def make_frame(cfg, seed):
    from paper_1604_03622_b200 import scenes
    p, q, n, D, G, ra, rb, K = cfg
    return scenes.bench_scene(p, q, n, seed=seed, movers=8).data[0]


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------- helpers
def fp64_peak_tflops():
    """Measured FP64 peak (tools/fp64_peak: DFMA and DMMA loops), best of both."""
    exe = os.path.join(ROOT, "tools", "fp64_peak")
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=60).stdout
        d = json.loads(out)
        return max(d["dfma_tflops"], d["dmma_m8n8k4_tflops"], d["dmma_m16n8k8_tflops"]), \
            "measured: tools/fp64_peak (max of DFMA / DMMA loops)"
    except Exception:
        return 37.2, "spec-derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz"


def ncu_traffic(name):
    path = os.path.join(ROOT, "profiles", name)
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    except (OSError, ValueError):
        return None, None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def fp64_roofline(flops, gram_ms):
    peak, peak_src = fp64_peak_tflops()
    traffic, _ = ncu_traffic("gram_ncu.json")
    achieved = flops / (gram_ms * 1e-3) / 1e12
    return {"kernel": "gram_herm_dmma (K1, sample covariance, FP64 DMMA engine)", "bound": "fp64",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": traffic,
            "algorithmic": f"4*n*(pq)^2 = {flops:.4e} flop per launch (8 flop per complex MAC, "
                           "Hermitian half)",
            "executed_tflops": 0.75 * achieved, "executed_frac": 0.75 * achieved / peak,
            "executed_note": "3M complex product: 6 real flop per complex MAC are executed",
            "peak_source": peak_src}


def int8_roofline(ops, gemm_ms, slices, flops, gram_ms):
    """Dominant kernel of the int8 engine: the slice GEMMs on the int8 tensor
    cores (int8 ops per Gram / GEMM span). Peak: 2 x the measured dense bf16
    rate in MEASURED_PEAKS.json (B200 int8 dense = 2 x bf16 dense)."""
    pk = measured_peaks()
    peak = 2.0 * pk.get("bf16_tflops_sustained", 1376.6)
    traffic, _ = ncu_traffic("gram_int8_ncu.json")
    achieved = ops / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else 0.0
    return {"kernel": f"int8 slice GEMMs of K1 (sample covariance, {slices} slices, tensor cores)",
            "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOP/s (int8)",
            "frac": achieved / peak, "traffic": traffic,
            "algorithmic": f"2*dpad^2*npad*3*s(s+1)/2 = {ops:.4e} int8 ops per Gram "
                           f"(exact slice products for the {flops:.4e}-flop complex Gram)",
            "gemm_span_ms": gemm_ms, "gram_stage_ms": gram_ms,
            "fp64_equivalent_tflops": flops / (gram_ms * 1e-3) / 1e12,
            "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops_sustained (int8 dense = 2 x bf16 "
                           "dense on B200); cuBLAS int8 measured 3.03 POPS here (tools/int8_probe.py)"}


def crt_roofline(nmod, n, d, tc_ms, executed_ops, flops, gram_ms):
    """Dominant kernel of the CRT engine: gram_tc_kernel (hand-written tcgen05,
    int8 tensor cores). Algorithmic work: per modulus four real int8 products
    (Re: XrXr + XiXi, Im: XiXr - XrXi) for each of the n d (d + 1) / 2 Hermitian
    entries, 2 ops per MAC. Duration: CUDA events bracketing that one launch
    (kst_stage_times entry 5). Peak: 2 x the measured dense bf16 rate in
    MEASURED_PEAKS.json (int8 dense = 2 x bf16 dense on B200)."""
    pk = measured_peaks()
    peak = 2.0 * pk.get("bf16_tflops_sustained", 1376.6)
    alg = 2.0 * 4.0 * nmod * n * d * (d + 1) / 2.0
    traffic, _ = ncu_traffic("gram_tc_ncu.json")
    achieved = alg / (tc_ms * 1e-3) / 1e12 if tc_ms > 0 else 0.0
    return {"kernel": f"gram_tc_kernel (K1 CRT Gram, {nmod} moduli, tcgen05 kind::i8, TMA, TMEM)",
            "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOP/s (int8)",
            "frac": achieved / peak, "traffic": traffic,
            "algorithmic": f"8*nmod*n*d(d+1)/2 = {alg:.4e} int8 ops per launch "
                           f"({executed_ops:.4e} issued incl. 128-tile padding)",
            "kernel_ms": tc_ms, "gram_stage_ms": gram_ms,
            "fp64_equivalent_tflops": flops / (gram_ms * 1e-3) / 1e12,
            "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops_sustained (int8 dense = 2 x bf16 "
                           "dense on B200)"}


def cpu_threads():
    return os.cpu_count() or 1


def oracle_frame(cube, cfg):
    from oracle import kron_oracle as orc
    p, q, n, D, G, ra, rb, K = cfg
    t0 = time.perf_counter()
    fit, ua, ub, vals = orc.pipeline(cube, ra, rb, D, G)
    return time.perf_counter() - t0, vals


# ----------------------------------------------------------------- reference arm
def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    cube = make_frame(cfg, 17)
    p, q, n, D, G, ra, rb, K = cfg
    px = n * D
    # bounded sample: each step is one full frame through the CPU port of the
    # reference path; the step count is capped so the run stays within minutes
    ksteps, wsteps = min(args.steps, 3), min(args.warmup, 1)
    for _ in range(wsteps):
        oracle_frame(cube, cfg)
    times = [oracle_frame(cube, cfg)[0] for _ in range(ksteps)]
    total = sum(times)
    value = px * ksteps / total
    line = {
        "impl": "reference", "metric": "STAP pixels/sec", "value": value, "unit": "pixels/s",
        "n_gpus": args.gpus, "steps": ksteps, "steps_requested": args.steps, "warmup": wsteps,
        "ms_per_step": 1e3 * total / ksteps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128/f64", "data": "synthetic (reference simulator, seed 17)",
        "config": config_block(args, cfg, world),
        "cpu_baseline": {"value": value, "unit": "pixels/s", "cores": cpu_threads(), "kind": "port",
                         "sample": f"{ksteps} full frame(s) through oracle/kron_oracle.pipeline "
                                   "(numpy restatement of the reference path; BLAS on all host threads)"},
        "e2e": {"value": value, "unit": "pixels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_block(args, cfg, world):
    p, q, n, D, G, ra, rb, K = cfg
    return {"workload": f"{args.config}: {n} range bins x {D} Doppler x {G} spatial, "
                        f"p={p} q={q}, ranks ({ra},{rb}), tol 1e-4, one frame per GPU per step",
            "p": p, "q": q, "n_bins": n, "D": D, "G": G, "rank_spatial": ra, "rank_temporal": rb,
            "frames_per_step": world, "parallelism": f"frame-sharded x{world}" if world > 1 else "single",
            "l2": "flushed (256 MB write) between timed steps; inputs (192 MB cube) exceed L2"}


# ----------------------------------------------------------------- our arm
def run_lmode(args, rank, local, world):
    """Supplementary line for configs[3] (L-mode windows): one
    256 x 256 frame per GPU per step through windowed_detection_image (n_w = 81
    training bins per test bin, ranks (1, 3)); N > 1 tiles ONE frame's test
    bins over the ranks (parallel.tile_bounds), each rank reading its tile plus
    the halo its windows reach, maps all-gathered over NCCL (strong scaling)."""
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_1604_03622_b200 as kst
    from paper_1604_03622_b200 import _native as nat
    p, q, nb, D, G, ra, rb, n_w = 3, 256, 256, 256, 16, 1, 3, 81
    from paper_1604_03622_b200 import parallel
    host = make_frame((p, q, nb, D, G, ra, rb, 1), 17)
    cube = torch.from_numpy(host).to(dev)
    lo, hi = parallel.tile_bounds(nb, world)[rank]
    dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
    c = nat.ctx(dev)
    for _ in range(args.warmup):
        kst.windowed_detection_image(cube, n_w, ra, rb, dop, grid, bins=(lo, hi))
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    l0 = nat.lib().kst_launch_count(c)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        kst.windowed_detection_image(cube, n_w, ra, rb, dop, grid, bins=(lo, hi))
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    launches = nat.lib().kst_launch_count(c) - l0
    # end to end: host cube in (this rank's tile + halo), full map gathered
    # over NCCL and copied to the host
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        full = parallel.windowed_sharded(host, n_w, ra, rb, dop, grid)
        full = full.cpu() if hasattr(full, "cpu") else full
    e2e_s = time.perf_counter() - t0
    a, b = kst.windowed.halo_range(lo, hi, n_w, nb)
    if world > 1:
        t = torch.tensor([ms, e2e_s * 1e3], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_s = float(t[0]), float(t[1]) / 1e3
    if rank != 0:
        return
    px = nb * D * args.steps
    base = None
    if not args.no_cpu_baseline:
        from oracle import kron_oracle as orc
        bins = list(range(0, nb, 32))
        tc = time.perf_counter()
        orc.windowed(host, n_w, ra, rb, D, G, bins=bins)
        tc = time.perf_counter() - tc
        base = {"value": len(bins) * D / tc, "unit": "pixels/s", "cores": cpu_threads(),
                "kind": "port",
                "sample": f"{len(bins)} test bins (one window estimate + detection each) of the "
                          f"same frame through oracle/kron_oracle.windowed"}
    print(json.dumps({
        "metric": "STAP pixels/sec", "value": px / (ms / 1e3), "unit": "pixels/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128/f64",
        "data": "synthetic (reference simulator restated in scenes.py; seeded, 8 movers)",
        "config": {"workload": f"configs[3] L-mode: {nb} bins x {D} Doppler x {G} spatial, p={p} "
                               f"q={q}, n_w={n_w} training bins per test bin "
                               f"({nb - n_w + 1} window estimates), ranks ({ra}, {rb})",
                   "parallelism": f"bin tiles + halo x{world}" if world > 1 else "single"},
        "e2e": {"value": px / e2e_s, "unit": "pixels/s",
                "h2d_bytes_per_step": int(host[a:b].nbytes),
                "d2h_bytes_per_step": int(nb * D * 8)},
        "gpu_launches": int(launches), "cpu_baseline": base,
        "roofline": None,
        "roofline_note": "latency-bound small per-window kernels (SURVEY.md §8d: no roofline for "
                         "the eigen stages); the frame headline is configs[1]"}))


def run_sweep(args, rank, local, world):
    """Supplementary line for configs[3]'s sweep (SURVEY.md §8 cfg 4): L-mode
    window n_w in {9, 25, 49, 81} (3x3 .. 9x9 training snapshots) x ranks
    (r_a, r_b) in {1, 2, 3}^2 on the 256 x 256 frame, plus the global
    estimate at each rank pair; 256-bin Doppler bank x 16 spatial steering
    candidates. One frame per point per step; value = all pixels of the
    sweep / its device time. r_a = p = 3 makes the map identically zero
    (SURVEY.md §8 window parity note): those points are timed and flagged.
    N > 1 runs the sweep on every rank (replicas)."""
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_1604_03622_b200 as kst
    p, q, nb, D, G = 3, 256, 256, 256, 16
    host = make_frame((p, q, nb, D, G, 1, 3, 1), 17 + rank)
    cube = torch.from_numpy(host).to(dev)
    dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
    points = [(n_w, ra, rb) for n_w in (9, 25, 49, 81, None) for ra in (1, 2, 3) for rb in (1, 2, 3)]

    def run(pt):
        n_w, ra, rb = pt
        if n_w is None:
            vals, _ = kst.process_frame_device(cube, ra, rb, dop, grid)
            return vals
        return kst.windowed_detection_image(cube, n_w, ra, rb, dop, grid).values

    for pt in points[: max(1, args.warmup)]:
        run(pt)
    rows, tot_ms = [], 0.0
    for pt in points:
        run(pt)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            v = run(pt)
        e1.record()
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / args.steps
        tot_ms += ms
        rows.append({"n_w": pt[0] or "global", "r_a": pt[1], "r_b": pt[2], "ms": ms,
                     "pixels_per_s": nb * D / (ms / 1e3),
                     "map_max": float(v.max()), "zero_map": pt[1] == p})
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t[0])
    if rank == 0:
        px = nb * D * len(points) * world
        print(json.dumps({
            "metric": "STAP pixels/sec", "value": px / (tot_ms / 1e3), "unit": "pixels/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128/f64",
            "data": "synthetic (reference simulator restated in scenes.py; seeded, 8 movers)",
            "config": {"workload": "configs[3] sweep: L-mode n_w in {9,25,49,81} + global, ranks "
                                   "(r_a, r_b) in {1,2,3}^2, 256 x 256 frame, 256 Doppler x 16 "
                                   "spatial; a step = the whole 45-point sweep",
                       "parallelism": "replicas" if world > 1 else "single"},
            "sweep": rows, "roofline": None,
            "roofline_note": "latency-bound per-window kernels; the frame headline is configs[1]"}),
            flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_multipass(args, rank, local, world):
    """Supplementary line for configs[4] (SURVEY.md §8 cfg 5): a 4-pass
    3-channel 2001 x 2001 stack per GPU per step, stacked to (n, 12, q),
    joint fit with ranks (K=4, 3) on the 24012 x 24012 covariance, one
    filtering and 4 pass maps (kst_pipeline with groups = 4). Pixels are
    pass-pixels (4 x n x D per frame). N > 1 runs independent stacks."""
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_1604_03622_b200 as kst
    from paper_1604_03622_b200 import _native as nat, scenes
    from paper_1604_03622_b200.pipeline import process_frame_device
    p, q, n, D, G, K, rb = 3, 2001, 2001, 2001, 16, 4, 3
    hist = scenes.bench_scene(p, q, n, seed=17 + rank, movers=8, n_passes=K)
    host = np.ascontiguousarray(kst.stack_passes(hist).data)  # (n, K p, q)
    host_pin = torch.from_numpy(host).pin_memory()
    cube = host_pin.to(dev)
    dop, grid = kst.make_doppler_grid(D), kst.make_stacked_spatial_grid(p, K, G)
    out = torch.empty((K, n, D), dtype=torch.float64, device=dev)
    c = nat.ctx(dev)
    for _ in range(args.warmup):
        process_frame_device(cube, K, rb, dop, grid, groups=K, out=out)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    st = torch.cuda.current_stream(dev)
    l0 = nat.lib().kst_launch_count(c)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        _, summ = process_frame_device(cube, K, rb, dop, grid, groups=K, out=out)
    e1.record(st)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    launches = nat.lib().kst_launch_count(c) - l0
    # end to end: pinned host stack -> HBM, pipeline, K maps -> pinned host,
    # every step; FrameStream overlaps stack i+1's upload and stack i-1's
    # maps download with stack i's compute
    from paper_1604_03622_b200.pipeline import FrameStream
    fs = FrameStream(tuple(host.shape), dev, K, rb, dop, grid, groups=K)
    fs.submit(host_pin)
    fs.flush()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fs.submit(host_pin)
    _, ev = fs.flush()
    ev.synchronize()
    torch.cuda.synchronize(dev)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([ms, e2e_s * 1e3], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_s = float(t[0]), float(t[1]) / 1e3
    if rank != 0:
        return
    px = K * n * D * world * args.steps
    base = None
    if not args.no_cpu_baseline:
        # bounded sample: the reference path on a q = 251 stack of the same
        # shape family (one full frame at q = 2001 needs a 9.2 GB S and ~2 min)
        from oracle import kron_oracle as orc
        qs = 251
        sm = scenes.bench_scene(p, qs, qs, seed=17, movers=2, n_passes=K)
        sd = orc.stack(sm.data)
        tc = time.perf_counter()
        fit = orc.lrkron(orc.scm(sd.reshape(qs, -1), K * p, qs), K * p, qs, K, rb)
        ua, ub = orc.filter_bases(fit)
        orc.pass_maps("kron", ua, ub, sd, K, p, orc.doppler_grid(qs), G)
        tc = time.perf_counter() - tc
        base = {"value": K * qs * qs / tc, "unit": "pixels/s", "cores": cpu_threads(),
                "kind": "port",
                "sample": f"one 4-pass stack at q = n_bins = D = {qs} through the oracle "
                          "(scm, lrkron, bases, pass_maps); pass-pixels/s"}
    print(json.dumps({
        "metric": "STAP pass-pixels/sec", "value": px / (ms / 1e3), "unit": "pixels/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128/f64",
        "data": "synthetic (reference simulator restated in scenes.py; 4 passes, seeded, 8 movers)",
        "config": {"workload": f"configs[4] multipass: K={K} passes x {n} bins x {D} Doppler, "
                               f"p={p} (stacked {K * p}) q={q}, ranks ({K}, {rb}), "
                               f"{G} spatial per pass; one stack per GPU per step",
                   "K": K, "p": p, "q": q, "n_bins": n, "D": D, "G": G,
                   "parallelism": "replicas" if world > 1 else "single",
                   "iterations": int(summ[0])},
        "e2e": {"value": px / e2e_s, "unit": "pixels/s",
                "h2d_bytes_per_step": int(host.nbytes), "d2h_bytes_per_step": int(K * n * D * 8)},
        "gpu_launches": int(launches), "cpu_baseline": base, "roofline": None,
        "roofline_note": "supplementary line; the roofline is reported on the configs[1] headline"}))


def main():
    args = parse()
    if args.config == "sweep" and args.impl == "ours":
        run_sweep(args, *dist_env())
        return
    if args.config == "lmode" and args.impl == "ours":
        run_lmode(args, *dist_env())
        return
    if args.config == "multipass" and args.impl == "ours":
        run_multipass(args, *dist_env())
        return
    cfg = CONFIGS[args.config]
    rank, local, world = dist_env()
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_1604_03622_b200 as kst
    from paper_1604_03622_b200 import _native as nat

    p, q, n, D, G, ra, rb, K = cfg
    seeds = [17, 18] if world == 1 else [1000 + rank, 1000 + world + rank]
    host_cubes = [make_frame(cfg, s) for s in seeds]
    cubes = [torch.from_numpy(c).to(dev) for c in host_cubes]
    dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
    out = torch.empty((1, n, D), dtype=torch.float64, device=dev)
    summ = np.zeros(8)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    c = nat.ctx(dev)
    lib = nat.lib()

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    def step(i):
        kst.process_frame_device(cubes[i % 2], ra, rb, dop, grid, out=out, summary=summ)

    for i in range(args.warmup):
        step(i)
    lib.kst_set_profiling(c, 1)
    clocks = ClockSampler(local)
    clocks.start()
    times, stages, iters = [], [], []
    launches0 = lib.kst_launch_count(c)
    for i in range(args.steps):
        flush.fill_(float(i))
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(i)
        e1.record(stream)
        barrier()
        times.append(e0.elapsed_time(e1))
        st = np.zeros(8)
        k = lib.kst_stage_times(c, st.ctypes.data_as(nat.C.c_void_p), 8)
        stages.append(st[:k].copy())
        iters.append(int(summ[0]))
    launches = lib.kst_launch_count(c) - launches0
    lib.kst_set_profiling(c, 0)

    # end to end through the public API with pinned host buffers: every step
    # copies its 192 MB cube host->device and its 32 MB map device->host;
    # FrameStream overlaps frame i+1's upload and frame i-1's download with
    # frame i's compute (upload, download and compute streams)
    from paper_1604_03622_b200.pipeline import FrameStream
    pinned = [torch.from_numpy(hc).pin_memory() for hc in host_cubes]
    # the PCIe bound of the end-to-end number: one pinned host->device cube copy
    probe = torch.empty(pinned[0].shape, dtype=pinned[0].dtype, device=dev)
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        h0.record(stream)
        probe.copy_(pinned[0], non_blocking=True)
        h1.record(stream)
    torch.cuda.synchronize(dev)
    h2d_ms = h0.elapsed_time(h1)
    del probe
    fs = FrameStream((n, p, q), dev, ra, rb, dop, grid)
    for i in range(args.warmup):
        fs.submit(pinned[i % 2])
    last = fs.flush()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fs.copy.wait_event(e0)
    for i in range(args.steps):
        fs.submit(pinned[i % 2])
    last = fs.flush()
    e1.record(fs.copy_back)  # after the final map reached the host
    barrier()
    torch.cuda.synchronize(dev)
    e2e_times = [e0.elapsed_time(e1)]
    clk = clocks.stop()

    tot = sum(times)
    e2e_tot = sum(e2e_times)
    if world > 1:
        t = torch.tensor([tot, e2e_tot], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot, e2e_tot = float(t[0]), float(t[1])
    px_step = n * D * world
    value = px_step * args.steps / (tot / 1e3)
    e2e_value = px_step * args.steps / (e2e_tot / 1e3)

    if rank == 0:
        st = np.mean(np.stack([np.pad(x, (0, 8 - len(x))) for x in stages]), axis=0)
        gram_ms = float(st[0])
        flops = 4.0 * n * float(p * q) ** 2          # Hermitian half, 8 flop per complex MAC
        engine, slices = kst.lrkron.get_gram_engine(dev)
        if engine == "int8":
            roof = int8_roofline(lib.kst_gram_int8_ops(c), float(st[5]), slices, flops, gram_ms)
        elif engine == "crt":
            roof = crt_roofline(slices, n, p * q, float(st[5]), lib.kst_gram_int8_ops(c), flops,
                                gram_ms)
        elif engine == "crt-cublas":
            roof = int8_roofline(lib.kst_gram_int8_ops(c), float(st[5]), slices, flops, gram_ms)
        else:
            roof = fp64_roofline(flops, gram_ms)
        line = {
            "metric": "STAP pixels/sec", "value": value, "unit": "pixels/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128/f64",
            "data": "synthetic (reference simulator restated in scenes.py; seeded SIRV clutter + 8 movers)",
            "config": config_block(args, cfg, world),
            "stages_ms": {"scm": gram_ms, "lrkron": float(st[1]), "bases": float(st[2]),
                          "detect": float(st[3])},
            "iterations": int(statistics.median(iters)),
            "gram_engine": {"mode": engine, "slices": slices},
            "roofline": roof,
            "e2e": {"value": e2e_value, "unit": "pixels/s",
                    "h2d_bytes_per_step": int(host_cubes[0].nbytes),
                    "d2h_bytes_per_step": int(n * D * 8),
                    "h2d_ms_per_cube": h2d_ms,
                    "h2d_gbps": host_cubes[0].nbytes / (h2d_ms * 1e-3) / 1e9,
                    "pcie_bound_pixels_per_s": px_step / (h2d_ms * 1e-3),
                    "note": "upload, compute and download overlap (FrameStream); the e2e "
                            "rate is bounded by the host->device copy of each 192 MB cube"},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if world == 1 and not args.no_cpu_baseline:
            oracle_frame(host_cubes[0][:64, :, :64].copy(), (p, 64, 64, 64, G, ra, rb, K))  # BLAS warm-up
            secs, ref_vals = oracle_frame(host_cubes[0], cfg)
            got = out[0].cpu().numpy()  # last step processed cubes[(steps-1) % 2]
            line["cpu_baseline"] = {
                "value": n * D / secs, "unit": "pixels/s", "cores": cpu_threads(), "kind": "port",
                "sample": "1 full frame through oracle/kron_oracle.pipeline (numpy restatement of "
                          "the reference path, BLAS on all host threads)"}
            del got, ref_vals
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
