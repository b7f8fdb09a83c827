"""Attribute an ncu SASS profile to CUDA source lines (via nvdisasm line info).

usage: python tools/sass_lines.py <report.ncu-rep> <lib.so> <kernel-substring>
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main(rep, lib, ksub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    cubins = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")]
    # function -> list of (offset, file, line)
    lines = {}
    for cb in cubins:
        out = subprocess.run(["nvdisasm", "-g", "-c", cb], capture_output=True, text=True).stdout
        fn, cur = None, None
        for ln in out.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln)
            if m:
                fn = m.group(1)
                lines[fn] = []
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
            if m and fn:
                lines[fn].append((int(m.group(1), 16), cur))
    cand = [f for f in lines if ksub in f]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "Kernel Name":
            if hdr is not None:
                break
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr:
            data.append(r)

    def f(x):
        try:
            return float(x.replace(",", ""))
        except Exception:
            return 0.0
    ie = hdr.index("Instructions Executed")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    base = int(data[0][0], 16)
    # pick the function whose instruction count matches
    best = None
    for fn in cand:
        if len(lines[fn]) == len(data):
            best = fn
    if best is None:
        best = min(cand, key=lambda fn: abs(len(lines[fn]) - len(data)))
    off2line = dict(lines[best])
    agg_i, agg_s = collections.Counter(), collections.Counter()
    for r in data:
        key = off2line.get(int(r[0], 16) - base)
        agg_i[key] += f(r[ie])
        agg_s[key] += f(r[si])
    ti, ts = sum(agg_i.values()) or 1, sum(agg_s.values()) or 1
    print(f"function {best}: {len(data)} sass, {ti:.0f} warp-inst, {ts:.0f} samples")
    for key, v in sorted(agg_i.items(), key=lambda kv: -kv[1])[:35]:
        print(f"  {str(key):40s} inst {v / ti * 100:5.1f}%  stall-samples {agg_s[key] / ts * 100:5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:4])
