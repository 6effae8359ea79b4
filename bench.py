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

# arithmetic of the path: c128 cube in, f64 map out; K1 (sample covariance)
# on the int8 tensor cores as an exact CRT integer Gram of the columns rounded
# to 32-bit significands (K1); K2-K5 in FP64
DTYPE = "f64 (K1: int8 CRT Gram of 32-bit-rounded columns)"

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
                    choices=sorted(CONFIGS) + ["lmode", "lmode-gotcha", "multipass", "sweep"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # internal: one threading mode of the reference arm (time_reference)
    ap.add_argument("--ref-worker", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--ref-threads", type=int, default=1, help=argparse.SUPPRESS)
    ap.add_argument("--ref-steps", type=int, default=3, help=argparse.SUPPRESS)
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


def int8_peak():
    """Measured dense int8 peak (profiles/r02_int8_peak.json, tools/int8_peak.py:
    cuBLASLt int8 8192^3 on this pool's B200, burst = best of 10 and sustained =
    4 s back to back). The bench's timed region is ~60 ms, so the BURST figure
    is the roofline denominator (B200_PROFILING.md: burst for a kernel timed
    alone or in a short region). Fallback: 2 x the measured bf16 burst."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_int8_peak.json")) as f:
            d = json.load(f)
        return (d["int8_dense_tops_burst"], d["int8_dense_tops_sustained"],
                "measured: cuBLASLt int8 8192^3 burst (best of 10), profiles/r02_int8_peak.json")
    except (OSError, ValueError, KeyError):
        pk = measured_peaks()
        b = 2.0 * pk.get("bf16_tflops", 1629.7)
        return b, 2.0 * pk.get("bf16_tflops_sustained", 1376.6), \
            "fallback: 2 x MEASURED_PEAKS.json bf16_tflops (burst)"


def crt_roofline(nmod, n, d, tc_ms, executed_ops, flops, gram_ms):
    """Dominant kernel of the CRT engine: gram_tc_kernel (hand-written tcgen05,
    int8 tensor cores). Algorithmic work: per modulus four real int8 products
    (Re: XrXr + XiXi, Im: XiXr - XrXi) for each of the n d (d + 1) / 2 Hermitian
    entries, 2 ops per MAC. Duration: CUDA events bracketing that one launch
    (kst_stage_times entry 5). Peak: the measured dense int8 rate in
    profiles/r02_int8_peak.json (burst; the sustained fraction is reported too)."""
    peak, peak_sus, peak_src = int8_peak()
    alg = 2.0 * 4.0 * nmod * n * d * (d + 1) / 2.0
    traffic, _ = ncu_traffic("gram_tc_ncu.json")
    achieved = alg / (tc_ms * 1e-3) / 1e12 if tc_ms > 0 else 0.0
    return {"kernel": f"gram_tc_kernel (K1 CRT Gram, {nmod} moduli, tcgen05 kind::i8, TMA, TMEM)",
            "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOP/s (int8)",
            "frac": achieved / peak, "traffic": traffic,
            "algorithmic": f"8*nmod*n*d(d+1)/2 = {alg:.4e} int8 ops per launch "
                           f"({executed_ops:.4e} issued incl. 128-tile padding)",
            "kernel_ms": tc_ms, "gram_stage_ms": gram_ms,
            "frac_of_sustained_peak": achieved / peak_sus, "peak_sustained": peak_sus,
            "fp64_equivalent_tflops": flops / (gram_ms * 1e-3) / 1e12,
            "peak_source": peak_src}


def cpu_threads():
    return os.cpu_count() or 1


def oracle_frame(cube, cfg):
    from oracle import kron_oracle as orc
    p, q, n, D, G, ra, rb, K = cfg
    t0 = time.perf_counter()
    fit, ua, ub, vals = orc.pipeline(cube, ra, rb, D, G)
    return time.perf_counter() - t0, vals


# ----------------------------------------------------------------- reference arm
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def host_info():
    """CPU model, core count, numpy and BLAS vendor/version of this host."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        import threadpoolctl
        info = [x for x in threadpoolctl.threadpool_info() if x.get("user_api") == "blas"]
        if info:
            blas = f"{info[0].get('internal_api')} {info[0].get('version')} ({info[0].get('architecture')})"
    except Exception:
        pass
    return {"cpu_model": model, "cores": cpu_threads(), "numpy": np.__version__, "blas": blas}


def ref_worker(args):
    """One threading mode of the reference arm, in its own process so the BLAS
    thread count is fixed before numpy loads (env set by the parent). Runs the
    UNMODIFIED reference package installed in baseline/_ref through its public
    API -- the README library sequence (pkg/README.md:144-161):
    sample_covariance -> lr_kron_estimate -> build_filter -> detection_image,
    with WorkerPool(threads) -- on the bench frame; one untimed warm-up on a
    small frame, then `steps` timed frames (perf_counter). Prints one JSON."""
    sys.path.insert(0, REF_DIR)
    import kronstap
    from kronstap.layout import cube_to_snapshots
    assert os.path.dirname(kronstap.__file__).startswith(REF_DIR), kronstap.__file__
    cfg = CONFIGS[args.config]
    p, q, n, D, G, ra, rb, K = cfg
    cube = make_frame(cfg, 17)
    dop, grid = kronstap.make_doppler_grid(D), kronstap.make_spatial_grid(p, G)

    def frame(c, pool, dd):
        scm = kronstap.sample_covariance(cube_to_snapshots(c), p, c.shape[2], pool=pool)
        est = kronstap.lr_kron_estimate(scm, ra, rb, pool=pool)
        filt = kronstap.build_filter("kron", estimate=est)
        return kronstap.detection_image(filt, c, dd, grid, pool=pool).values

    with kronstap.WorkerPool(args.ref_threads) as pool:
        small = np.ascontiguousarray(cube[:96, :, :64])
        frame(small, pool, kronstap.make_doppler_grid(64))  # warm-up (BLAS threads, page-in)
        times = []
        for _ in range(args.ref_steps):
            t0 = time.perf_counter()
            vals = frame(cube, pool, dop)
            times.append(time.perf_counter() - t0)
    print(json.dumps({"times": times, "map_sum": float(vals.sum()),
                      "kronstap": os.path.dirname(kronstap.__file__)}), flush=True)


def time_reference(args, steps, modes=("blas", "pool")):
    """Time the reference on this host in the SURVEY.md §8(d) threading modes:
    "blas" = OPENBLAS_NUM_THREADS=N with WorkerPool(1); "pool" =
    OPENBLAS_NUM_THREADS=1 with WorkerPool(N) (src/parallel.py:34-68). Each
    mode runs in a subprocess. Returns {mode: median seconds per frame} and
    the per-mode records, or None when baseline/_ref is absent."""
    if not os.path.isdir(os.path.join(REF_DIR, "kronstap")):
        return None
    ncore = cpu_threads()
    out = {}
    for mode in modes:
        env = dict(os.environ)
        blas_t, pool_t = (ncore, 1) if mode == "blas" else (1, ncore)
        for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
            env[k] = str(blas_t)
        env.pop("RANK", None), env.pop("WORLD_SIZE", None), env.pop("LOCAL_RANK", None)
        cmd = [sys.executable, os.path.abspath(__file__), "--config", args.config, "--ref-worker",
               "--ref-threads", str(pool_t), "--ref-steps", str(steps)]
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1800)
        if r.returncode != 0:
            out[mode] = {"error": r.stderr.strip().splitlines()[-1:] if r.stderr else "rc != 0"}
            continue
        rec = json.loads(r.stdout.strip().splitlines()[-1])
        rec["median_s"] = statistics.median(rec["times"])
        rec["blas_threads"], rec["pool_threads"] = blas_t, pool_t
        out[mode] = rec
    return out


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    p, q, n, D, G, ra, rb, K = cfg
    px = n * D
    # bounded sample: each timed step is one full frame through the reference;
    # at most 3 timed frames per threading mode so the arm ends within minutes
    ksteps = max(1, min(args.steps, 3))
    modes = time_reference(args, ksteps)
    if modes and any("median_s" in m for m in modes.values()):
        ok = {k: v for k, v in modes.items() if "median_s" in v}
        best = min(ok, key=lambda k: ok[k]["median_s"])
        secs = ok[best]["median_s"]
        kind = "reference"
        sample = (f"median of {ksteps} full frames per threading mode through the unmodified "
                  f"reference (baseline/_ref/kronstap, README library sequence); faster mode "
                  f"'{best}' reported")
        cores = ok[best]["blas_threads"] * ok[best]["pool_threads"]
        detail = {k: {kk: v[kk] for kk in ("median_s", "times", "blas_threads", "pool_threads")
                      if kk in v} if "median_s" in v else v for k, v in modes.items()}
    else:
        # reference not installed: the numpy restatement (oracle port)
        cube = make_frame(cfg, 17)
        oracle_frame(np.ascontiguousarray(cube[:64, :, :64]), (p, 64, 64, 64, G, ra, rb, K))
        ts = [oracle_frame(cube, cfg)[0] for _ in range(ksteps)]
        secs, kind, cores, detail = statistics.median(ts), "port", cpu_threads(), None
        sample = f"median of {ksteps} full frames through oracle/kron_oracle.pipeline"
    value = px / secs
    line = {
        "impl": "reference", "metric": "STAP pixels/sec", "value": value, "unit": "pixels/s",
        "n_gpus": args.gpus, "steps": ksteps, "steps_requested": args.steps, "warmup": 1,
        "ms_per_step": 1e3 * secs, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128/f64", "data": "synthetic (reference simulator, seed 17)",
        "config": config_block(args, cfg, world),
        "cpu_baseline": {"value": value, "unit": "pixels/s", "cores": cores, "kind": kind,
                         "sample": sample, "modes": detail, "host": host_info()},
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
    256 x 256 frame (--config lmode) or one Gotcha-scale 2001 x 2001 frame
    (--config lmode-gotcha) per GPU per step through windowed_detection_image
    (n_w = 81 training bins per test bin, ranks (1, 3)); N > 1 tiles ONE frame's test
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
    gotcha = args.config == "lmode-gotcha"
    p, q, nb, D, G, ra, rb, n_w = (3, 2001, 2001, 2001, 16, 1, 3, 81) if gotcha else \
        (3, 256, 256, 256, 16, 1, 3, 81)
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
    winfo = kst.windowed.last_window_info()
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
        # bounded sample: a few interior test bins, each its own window
        # estimate + detection (~9 s per window at Gotcha scale)
        bins = [nb // 3, nb // 2] if gotcha else list(range(0, nb, 32))
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
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": DTYPE,
        "data": "synthetic (reference simulator restated in scenes.py; seeded, 8 movers)",
        "config": {"workload": f"configs[3] L-mode{' at Gotcha scale' if gotcha else ''}: "
                               f"{nb} bins x {D} Doppler x {G} spatial, p={p} "
                               f"q={q}, n_w={n_w} training bins per test bin "
                               f"({nb - n_w + 1} window estimates), ranks ({ra}, {rb})",
                   "parallelism": f"bin tiles + halo x{world}" if world > 1 else "single"},
        "e2e": {"value": px / e2e_s, "unit": "pixels/s",
                "h2d_bytes_per_step": int(host[a:b].nbytes),
                "d2h_bytes_per_step": int(nb * D * 8)},
        "gpu_launches": int(launches), "cpu_baseline": base,
        "window_info": {"fallback_windows": int(np.sum(winfo[:, 0] == 64)) if winfo is not None
                        else None,
                        "max_rayleigh_ritz_rounds": int(winfo[:, 5].max()) if winfo is not None
                        else None},
        "roofline": None,
        "roofline_note": "per-window eigensolves are latency chains (SURVEY.md §8d: no roofline "
                         "for the eigen stages); kernel split in profiles/; the frame headline is "
                         "configs[1]"}))


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
            "vs_baseline": None, "dtype": DTYPE,
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
        "vs_baseline": None, "dtype": DTYPE,
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
    if args.ref_worker:
        ref_worker(args)
        return
    if args.config == "sweep" and args.impl == "ours":
        run_sweep(args, *dist_env())
        return
    if args.config in ("lmode", "lmode-gotcha") and args.impl == "ours":
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
        # communicator logging (rank count visible to the driver)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
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

    # The frame as a CUDA graph (FrameGraph: kst_pipeline_async captured once
    # per cube buffer, one graph launch per frame, every decision on the
    # device); KST_BENCH_GRAPH=0 times the direct kst_pipeline call instead.
    # Profiling is on before the capture, so the stage marks are event-record
    # nodes of the graph and every replay re-times its stages.
    use_graph = os.environ.get("KST_BENCH_GRAPH", "1") != "0"
    lib.kst_set_profiling(c, 1)
    graphs = []
    if use_graph:
        from paper_1604_03622_b200.pipeline import FrameGraph
        graphs = [FrameGraph(cb, ra, rb, dop, grid, out=out) for cb in cubes]

    def step(i):
        if use_graph:
            graphs[i % 2].replay()
        else:
            kst.process_frame_device(cubes[i % 2], ra, rb, dop, grid, out=out, summary=summ)

    try:
        for i in range(args.warmup):
            step(i)
    except Exception as exc:  # capture refused (driver / runtime): time the direct call
        if not use_graph:
            raise
        print(f"bench: CUDA-graph capture failed ({exc}); timing the direct kst_pipeline call",
              file=sys.stderr)
        torch.cuda.synchronize(dev)
        use_graph = False
        for i in range(args.warmup):
            step(i)
    clocks = ClockSampler(local)
    clocks.start()

    def timed_steps():
        """K timed steps; None when a replayed frame left the sync-free form
        (its values would come from the synchronous recomputation, outside
        the timed graph) -- the caller then times the direct call."""
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
            if use_graph:  # the device outcome record of this replay (ok, iterations, ...)
                rec = graphs[i % 2].rec.cpu().numpy()
                if rec[0] != 1.0:
                    return None
                iters.append(int(rec[1]))
            else:
                iters.append(int(summ[0]))
        launches = lib.kst_launch_count(c) - launches0
        if use_graph:  # host-side count is 0 for replays: kernels per captured frame
            launches = sum(graphs[i % 2].launches for i in range(args.steps))
        return times, stages, iters, launches

    res = timed_steps()
    if res is None:
        print("bench: a replayed frame left the sync-free form; timing the direct call",
              file=sys.stderr)
        use_graph = False
        for i in range(args.warmup):
            step(i)
        res = timed_steps()
    times, stages, iters, launches = res
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
    # N > 1: every step's maps are all-gathered over NCCL (NVLink) and rank 0
    # downloads the gathered stack -- the map gather is inside the e2e region
    fs = FrameStream((n, p, q), dev, ra, rb, dop, grid,
                     gather_group=dist.group.WORLD if world > 1 else None)
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
    # the numpy drop-in call a reference user makes (kst.process_frame on a
    # pageable numpy cube -> numpy map): staged upload, compute, staged
    # download, frames back to back (no cross-frame overlap); host wall clock
    numpy_api = None
    if world == 1:
        for i in range(2):
            kst.process_frame(host_cubes[i % 2], ra, rb, dopplers=dop, spatial_grid=grid)
        nk = max(3, min(args.steps, 6))
        t0 = time.perf_counter()
        for i in range(nk):
            vals_np, _ = kst.process_frame(host_cubes[i % 2], ra, rb, dopplers=dop, spatial_grid=grid)
        secs = (time.perf_counter() - t0) / nk
        numpy_api = {"value": n * D / secs, "unit": "pixels/s", "ms_per_frame": secs * 1e3,
                     "frames": nk,
                     "note": "kst.process_frame(numpy cube) -> numpy map, pageable host memory "
                             "(kst_copy_staged through pinned chunks), frames back to back"}

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
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": DTYPE,
            "data": "synthetic (reference simulator restated in scenes.py; seeded SIRV clutter + 8 movers)",
            "config": config_block(args, cfg, world),
            "stages_ms": {"scm": gram_ms, "lrkron": float(st[1]), "bases": float(st[2]),
                          "detect": float(st[3])},
            "iterations": int(statistics.median(iters)),
            "gram_engine": {"mode": engine, "slices": slices},
            "roofline": roof,
            "e2e": {"value": e2e_value, "unit": "pixels/s",
                    "h2d_bytes_per_step": int(host_cubes[0].nbytes),
                    "d2h_bytes_per_step": int(world * n * D * 8),
                    "nccl_gather_bytes_per_step": int((world - 1) * world * n * D * 8)
                    if world > 1 else 0,
                    "h2d_ms_per_cube": h2d_ms,
                    "h2d_gbps": host_cubes[0].nbytes / (h2d_ms * 1e-3) / 1e9,
                    "pcie_bound_pixels_per_s": px_step / (h2d_ms * 1e-3),
                    "note": "upload, compute and download overlap (FrameStream); the e2e "
                            "rate is bounded by the host->device copy of each 192 MB cube"
                            + ("; N > 1: each step's maps all-gathered over NCCL and the "
                               "gathered stack read back by rank 0" if world > 1 else "")},
            "gpu_launches": int(launches),
            "frame_api": ("FrameGraph: kst_pipeline_async captured as one CUDA graph per cube "
                          "buffer, one graph launch per frame" if use_graph else
                          "process_frame_device (kst_pipeline, one host sync per frame)"),
            "clocks": clk,
        }
        if numpy_api is not None:
            line["e2e"]["numpy_api"] = numpy_api
        if world == 1 and not args.no_cpu_baseline:
            # bounded sample: the unmodified reference (baseline/_ref) in its
            # faster threading mode (BLAS threads), median of 2 full frames
            modes = time_reference(args, 2, modes=("blas",))
            if modes and "median_s" in modes.get("blas", {}):
                m = modes["blas"]
                line["cpu_baseline"] = {
                    "value": n * D / m["median_s"], "unit": "pixels/s",
                    "cores": m["blas_threads"] * m["pool_threads"], "kind": "reference",
                    "sample": "median of 2 full frames through the unmodified reference "
                              "(baseline/_ref/kronstap, README library sequence, "
                              "OPENBLAS_NUM_THREADS = all host cores, WorkerPool(1))",
                    "host": host_info()}
            else:
                secs, _ = oracle_frame(host_cubes[0], cfg)
                line["cpu_baseline"] = {
                    "value": n * D / secs, "unit": "pixels/s", "cores": cpu_threads(),
                    "kind": "port",
                    "sample": "1 full frame through oracle/kron_oracle.pipeline (numpy "
                              "restatement of the reference path, BLAS on all host threads)",
                    "host": host_info()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
