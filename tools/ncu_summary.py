"""Summarise an ncu report: key details + top SASS stall sites (run here, no GPU)."""
import csv
import io
import subprocess
import sys


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    keys = ("Duration", "DRAM Throughput", "Memory Throughput", "Registers Per Thread",
            "Achieved Occupancy", "Theoretical Occupancy", "Compute (SM) Throughput",
            "L2 Cache Throughput", "Block Size", "Grid Size", "Executed Ipc Active",
            "Warp Cycles Per Issued Instruction", "Elapsed Cycles", "L1/TEX Hit Rate", "L2 Hit Rate")
    seen = set()
    for line in out.splitlines():
        s = line.strip()
        for k in keys:
            if s.startswith(k) and k not in seen:
                seen.add(k)
                print("  ", s)


def raw(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {}
    for n in names:
        if n in hdr:
            i = hdr.index(n)
            res[n] = (vals[i], units[i])
    return res


def sass(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = []
            blocks.append(cur)
            continue
        if cur is not None:
            cur.append(r)
    hdr, data = blocks[0][0], blocks[0][1:]

    def f(x):
        try:
            return float(x.replace(",", ""))
        except Exception:
            return 0.0
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    tot = sum(f(r[si]) for r in data) or 1
    print(f"  samples {tot:.0f}, warp-instructions executed {sum(f(r[ie]) for r in data):.0f}")
    sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    agg = {}
    for r in data:
        for i in sc:
            agg[hdr[i][6:]] = agg.get(hdr[i][6:], 0) + f(r[i])
    print("  stalls:", ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    # opcode mix by executed count
    mix = {}
    for r in data:
        op = r[1].split()[0] if r[1] else "?"
        if op.startswith("@"):
            op = r[1].split()[1]
        op = op.split(".")[0]
        mix[op] = mix.get(op, 0) + f(r[ie])
    tot_i = sum(mix.values()) or 1
    print("  mix:", ", ".join(f"{k} {v / tot_i * 100:.0f}%" for k, v in sorted(mix.items(), key=lambda x: -x[1])[:14]))
    for r in sorted(data, key=lambda r: -f(r[si]))[:top]:
        st = sorted(((f(r[i]), hdr[i][6:]) for i in sc), reverse=True)[:2]
        print(f"   {f(r[si]) / tot * 100:5.1f}%  {r[1][:64]:64s} {st}")


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print("==", rep)
        details(rep)
        for k, v in raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                              "gpu__time_duration.sum", "sm__inst_executed.sum"]).items():
            print("  ", k, v)
        sass(rep)
