"""Per-kernel roofline table of one Gotcha frame from an `ncu --set full` report.

  ncu --set full --clock-control none -o rep python tools/one_frame.py 2001 1
  python tools/roofline_table.py rep.ncu-rep > profiles/r01_kernel_roofline.md

For every kernel: ncu duration, DRAM bytes (read + write), DRAM bandwidth as
a fraction of MEASURED_PEAKS.json hbm_gbs, pipe activity (tensor / FP64 /
ALU), achieved occupancy, and -- where SURVEY.md §8d / DESIGN.md §4 define
the algorithmic work of the kernel -- the algorithmic rate against its peak.
ncu times are serialised and cold-cache (clock control off); the bench line
measures the same kernels warm inside the frame.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N, P, Q, D, NMOD = 2001, 3, 2001, 2001, 10
DIM = P * Q
C128 = 16
PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
HBM = PEAKS.get("hbm_gbs", 6548.8) * 1e9
_I8 = os.path.join(ROOT, "profiles", "r02_int8_peak.json")
# measured int8 dense burst peak (cuBLASLt, profiles/r02_int8_peak.json); else 2 x bf16
INT8 = (json.load(open(_I8))["int8_dense_tops_burst"] * 1e12 if os.path.exists(_I8)
        else 2.0 * PEAKS.get("bf16_tflops", 1608.5) * 1e12)
FP64 = 37.0e12  # B200 FP64 (vector / DMMA) nominal; tools/fp64_peak measures it on the box

# algorithmic work per launch: (kind, amount, note)
ALG = {
    "gram_tc_kernel": ("int8", 8.0 * NMOD * N * DIM * (DIM + 1) / 2,
                       "8 N n d(d+1)/2 int8 ops (exact CRT products)"),
    "crt_residue_kernel": ("bytes", N * DIM * C128 + DIM * NMOD * 2 * 2016,
                           "cube read + residues written"),
    "colmax_split_kernel": ("bytes", N * DIM * C128, "cube read"),
    "crt_strip_combine_kernel": ("bytes", 1128 * NMOD * 2 * 128 * 128 + DIM * DIM * C128,
                                 "residue tiles read + S written"),
    "mgram_split_kernel": ("bytes", DIM * DIM * C128, "S read once"),
    "bstep_kernel": ("bytes", DIM * DIM * C128, "S read once"),
    "bz2_kernel": ("bytes", Q * Q * C128, "b read once"),
    "detect_bin_kernel": ("bytes", N * DIM * C128 + N * D * 8, "cube read + map written (HBM); "
                          "FP64-issue bound, DESIGN.md §4 K5"),
    "detect_f32_kernel": ("bytes", N * DIM * C128 + N * D * 8, "cube read + map written (HBM); "
                          "FP32 transform issue/latency bound, DESIGN.md §4 K5"),
}


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {k: hdr.index(k) for k in hdr}

    def val(r, m, scale=None):
        if m not in col:
            return None
        try:
            v = float(r[col[m]].replace(",", ""))
        except ValueError:
            return None
        u = units[col[m]]
        if scale == "time":
            v *= {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3,
                  "ms": 1e-3, "second": 1.0, "s": 1.0}[u]
        if scale == "bytes":
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3,
                  "MB": 1e6, "GB": 1e9}[u]
        return v

    agg = {}
    order = []
    for r in rows[2:]:
        name = re.sub(r"\(.*", "", r[col["Kernel Name"]]).split("::")[-1].split("<")[0].strip()
        t = val(r, "gpu__time_duration.sum", "time") or 0.0
        rd = val(r, "dram__bytes_read.sum", "bytes") or 0.0
        wr = val(r, "dram__bytes_write.sum", "bytes") or 0.0
        pipes = [val(r, m) or 0.0 for m in (
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active")]
        a = agg.setdefault(name, [0, 0.0, 0.0, [0.0] * 4])
        if name not in order:
            order.append(name)
        a[0] += 1
        a[1] += t
        a[2] += rd + wr
        a[3] = [x + y * t for x, y in zip(a[3], pipes)]
    total = sum(a[1] for a in agg.values())
    print(f"# Per-kernel roofline, one Gotcha frame (ncu --set full, cold, serialised)\n")
    print(f"HBM peak {HBM / 1e12:.2f} TB/s, int8 dense peak {INT8 / 1e12:.0f} TOP/s "
          f"(profiles/r02_int8_peak.json, MEASURED_PEAKS.json); frame total {total * 1e6:.0f} us over {len(order)} kernels.\n")
    print("| kernel | calls | us | share | DRAM MB | DRAM TB/s | frac HBM | tensor % | FP64 % "
          "| ALU % | warps % | algorithmic rate | frac of its peak |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for name in sorted(order, key=lambda k: -agg[k][1]):
        c, t, b, pw = agg[name]
        pw = [x / t if t else 0.0 for x in pw]
        bw = b / t if t else 0.0
        alg, frac = "", ""
        if name in ALG:
            kind, amt, note = ALG[name]
            per = t / c
            if kind == "int8":
                rate = amt / per
                alg, frac = f"{rate / 1e12:.0f} TOP/s ({note})", f"{rate / INT8:.2f}"
            else:
                rate = amt / per
                alg, frac = f"{rate / 1e12:.2f} TB/s ({note})", f"{rate / HBM:.2f}"
        print(f"| {name} | {c} | {t * 1e6:.1f} | {100 * t / total:.1f}% | {b / 1e6:.0f} | "
              f"{bw / 1e12:.2f} | {bw / HBM:.2f} | {pw[0]:.0f} | {pw[1]:.0f} | {pw[2]:.0f} | "
              f"{pw[3]:.0f} | {alg} | {frac} |")


if __name__ == "__main__":
    main()
