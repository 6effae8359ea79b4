"""Dense int8 tensor-core peak of this B200, by the MEASURED_PEAKS.json recipe:
cuBLASLt int8 GEMM (torch._int_mm, int32 accumulate) at m = n = k = 8192,
2*m*n*k ops per call; burst = best of 10 single calls (CUDA events), sustained
= back to back for 4 s. The dense bf16 rate is re-measured the same way in the
same process so the two share clocks and power state. Output: one JSON object
(profiles/r02_int8_peak.json), used by bench.py as the roofline denominator of
the int8 Gram kernel.

    python tools/int8_peak.py > profiles/r02_int8_peak.json
"""
import json
import subprocess
import threading
import time

import torch


def _smi(stop, out):
    while not stop.is_set():
        try:
            r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                                "--format=csv,noheader,nounits"], capture_output=True,
                               text=True, timeout=5)
            mhz, w = r.stdout.strip().splitlines()[0].split(",")
            out.append((float(mhz), float(w)))
        except Exception:
            pass
        time.sleep(0.2)


def rate(fn, ops, burst_reps=10, sustain_s=4.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(burst_reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    stop, samples = threading.Event(), []
    th = threading.Thread(target=_smi, args=(stop, samples), daemon=True)
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    calls, t_end = 0, time.perf_counter() + sustain_s
    e0.record()
    while time.perf_counter() < t_end:
        for _ in range(8):
            fn()
        calls += 8
        torch.cuda.synchronize() if calls % 64 == 0 else None
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    sus_ms = e0.elapsed_time(e1)
    mhz = sorted(s[0] for s in samples)
    return {"burst_tops": ops / (best * 1e-3) / 1e12,
            "sustained_tops": ops * calls / (sus_ms * 1e-3) / 1e12,
            "calls": calls, "sm_mhz_median": mhz[len(mhz) // 2] if mhz else None,
            "power_w_max": max((s[1] for s in samples), default=None)}


def main():
    dev = torch.device("cuda", 0)
    m = n = k = 8192
    a = torch.randint(-127, 128, (m, k), dtype=torch.int8, device=dev)
    b = torch.randint(-127, 128, (n, k), dtype=torch.int8, device=dev).t()  # column-major B
    i8 = rate(lambda: torch._int_mm(a, b), 2.0 * m * n * k)
    a16 = torch.randn(m, k, dtype=torch.bfloat16, device=dev)
    b16 = torch.randn(k, n, dtype=torch.bfloat16, device=dev)
    bf = rate(lambda: a16 @ b16, 2.0 * m * n * k)
    print(json.dumps({
        "gpu": torch.cuda.get_device_name(0),
        "how": "torch._int_mm int8 8192^3 (cuBLASLt, int32 accumulate) and torch.matmul bf16 8192^3; "
               "2*m*n*k ops; burst = best of 10 (CUDA events), sustained = back to back for 4 s",
        "int8_dense_tops_burst": i8["burst_tops"], "int8_dense_tops_sustained": i8["sustained_tops"],
        "bf16_dense_tflops_burst": bf["burst_tops"], "bf16_dense_tflops_sustained": bf["sustained_tops"],
        "int8": i8, "bf16": bf}, indent=1))


if __name__ == "__main__":
    main()
