#!/usr/bin/env python
"""Attribute ncu per-SASS-instruction counters to CUDA source lines.

    python tools/sass_lines.py <report.ncu-rep> <kernel-mangled-name> <lib.so> [metric]

Uses nvdisasm -g line info of the kernel's cubin (built with -lineinfo) and
`ncu --page source --print-source sass` counters; prints the top lines.
"""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path


def main():
    rep, kern, lib = sys.argv[1:4]
    lib = str(Path(lib).resolve())
    metric = sys.argv[4] if len(sys.argv) > 4 else "Instructions Executed"
    tmp = Path(tempfile.mkdtemp())
    subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
    where = {}
    for cub in tmp.glob("*.cubin"):
        txt = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout
        sec = re.search(r"\.text\." + re.escape(kern) + r":\n(.*?)(?=\n\s*\.section|\Z)", txt, re.S)
        if not sec:
            continue
        cur = None
        for line in sec.group(1).splitlines():
            m = re.search(r'//## File "([^"]+)", line (\d+)', line)
            if m:
                cur = (Path(m.group(1)).name, int(m.group(2)))
                continue
            a = re.match(r"\s*/\*([0-9a-f]{4,})\*/", line)
            if a and cur:
                where[int(a.group(1), 16)] = cur
        break
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    addrs = []
    for r in rows[hdr + 1:]:
        try:
            addrs.append(int(r[0], 16))
        except (ValueError, IndexError):
            pass
    base = min(addrs) if addrs else 0
    agg = collections.Counter()
    stall = collections.Counter()
    tot = 0
    for r in rows[hdr + 1:]:
        d = dict(zip(h, r))
        try:
            addr = int(d["Address"], 16) - base
            v = float(d.get(metric, "0") or 0)
            s = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except (ValueError, KeyError):
            continue
        key = where.get(addr, ("?", 0))
        agg[key] += v
        stall[key] += s
        tot += v
    ts = sum(stall.values()) or 1
    print(f"total {metric}: {tot:.4g}")
    for (f, l), v in sorted(agg.items(), key=lambda kv: -stall[kv[0]])[:int(__import__("os").environ.get("TOPN","45"))]:
        print(f"{f}:{l:<5d} instr {100 * v / tot:5.1f}%   stall-samples {100 * stall[(f, l)] / ts:5.1f}%")


if __name__ == "__main__":
    main()
