"""Summarise one kernel of an ncu --set full report into a profiles/*.json.

  python tools/ncu_summary.py REPORT.ncu-rep KERNEL_REGEX OUT.json "description"

Keeps the figures bench.py and DESIGN.md cite: duration, DRAM bytes read and
written (the roofline `traffic`), tensor / FP64 / ALU pipe activity, L2 and
DRAM throughput, achieved occupancy and registers.
"""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-3),
    "dram_bytes_read": ("dram__bytes_read.sum", None),
    "dram_bytes_write": ("dram__bytes_write.sum", None),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "fp64_pipe_active_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "alu_pipe_active_pct": ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "l2_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "dram_throughput_pct": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "registers_per_thread": ("launch__registers_per_thread", 1),
    "grid_size": ("launch__grid_size", 1),
    "block_size": ("launch__block_size", 1),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
        "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}


def main():
    rep, kre, out, desc = sys.argv[1:5]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    sel = [r for r in rows[2:] if re.search(kre, r[hdr.index("Kernel Name")])]
    if not sel:
        raise SystemExit(f"no kernel matching {kre!r}")
    r = sel[-1]
    res = {"kernel": r[hdr.index("Kernel Name")][:160], "source": desc, "launches_in_report": len(sel)}
    for k, (m, _) in KEYS.items():
        if m not in hdr:
            continue
        i = hdr.index(m)
        try:
            v = float(r[i].replace(",", ""))
        except ValueError:
            continue
        u = units[i]
        if k == "duration_ms":
            v = v * UNIT.get(u, 1.0) * 1e3
        elif k.startswith("dram_bytes"):
            v = v * UNIT.get(u, 1.0)
        res[k] = v
    if "dram_bytes_read" in res and "dram_bytes_write" in res:
        res["dram_bytes_per_launch"] = res["dram_bytes_read"] + res["dram_bytes_write"]
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
