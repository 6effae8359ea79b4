"""Attribute ncu warp-stall samples to CUDA source lines.

  ncu -i rep --page source --csv --kernel-name regex:K --launch-count 1 > sass.csv
  nvdisasm -g -c lib.cubin > all.sass        (cubin from cuobjdump -xelf all lib.so)
  python tools/sass_lines.py sass.csv all.sass KERNEL_SUBSTRING [top]

The ncu SASS page lists absolute addresses; offsets are taken relative to the
first row (the function entry), matched to the `/*offset*/` lines of the
nvdisasm listing of the function whose name contains KERNEL_SUBSTRING, and
the samples are summed per `//## File ..., line N` annotation.
"""
import collections
import csv
import re
import sys


def sass_offsets(path, kname):
    lines = open(path).read().splitlines()
    start = None
    for i, l in enumerate(lines):
        if l.startswith(".text.") and kname in l:
            start = i
            break
    if start is None:
        raise SystemExit(f"function containing {kname!r} not found")
    cur = None
    off2line = {}
    for l in lines[start + 1:]:
        if l.startswith(".text."):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m:
            off2line[int(m.group(1), 16)] = cur
    return off2line


def main():
    csv_path, sass_path, kname = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    rows = list(csv.reader(open(csv_path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_e = hdr.index("Instructions Executed")
    data = []
    for r in rows[hdr_i + 1:]:
        if not r or not r[0].startswith("0x"):
            break  # first function only
        data.append((int(r[0], 16), int(r[i_s] or 0), int(r[i_e] or 0)))
    base = data[0][0]
    off2line = sass_offsets(sass_path, kname)
    samp = collections.Counter()
    inst = collections.Counter()
    for addr, s, e in data:
        key = off2line.get(addr - base, "?")
        samp[key] += s
        inst[key] += e
    tot = sum(samp.values()) or 1
    print(f"{'line':24s} {'samples':>8s} {'share':>6s} {'warp-inst':>10s}")
    for k, v in samp.most_common(top):
        print(f"{k:24s} {v:8d} {100 * v / tot:5.1f}% {inst[k]:10d}")


if __name__ == "__main__":
    main()
