"""Small driver for ncu: one engine, a few device solves (no timing claims)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1209_4297_b200 import engine as E  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--order", type=int, default=1)
ap.add_argument("--nt", type=int, default=200)
ap.add_argument("--points", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--resident", action="store_true", help="resident march on segmented lines (levels == 1)")
a = ap.parse_args()
sysm, nt, cfg = bench.workload(a.workload, a.points or None, None)
full_nt = nt
nt = a.nt or nt
# keep the workload's dt (and hence the stiffness r and the solve geometry): shorten T instead
from paper_1209_4297_b200 import problems as P  # noqa: E402
ivp = sysm.ivp
sysm = P.StructuredIVP(ivp.problem, ivp.t_start, ivp.t_start + (ivp.t_end - ivp.t_start) * nt / full_nt,
                       ivp.initial_state)
eng = E.Engine(sysm, E.RidcConfig(levels=a.order, steps=nt), resident_segments=a.resident)
y0 = torch.from_numpy(np.array(sysm.initial_state)).cuda()
out = torch.empty_like(y0)
for _ in range(a.reps):
    t = eng.run_device(y0, out)
print(f"{cfg['workload']} p={a.order} nt={nt}: {t*1e3:.3f} ms/solve, {t/ (nt + a.order*(a.order-1)//2)*1e6:.2f} us/tick", eng.info)
if os.environ.get("RIDC_PHASE_TIMING"):
    import ctypes
    from paper_1209_4297_b200 import _lib
    buf = (ctypes.c_longlong * (128 + 4096))()
    _lib.check(_lib.lib().ridc_debug_phase_trace(eng._h, buf, 128 + 4096))
    names = ["start", "node0", "accum", "stencil", "fwd", "scan1", "carry+bwd", "scan2", "store0", "end"]
    for it in range(8):
        st = [buf[it * 16 + k] for k in range(10)]
        if st[0] == 0:
            break
        d = [st[k] - st[k - 1] for k in range(1, 10)]
        print(f"item {it}: " + " ".join(f"{names[k]}:{d[k-1]}" for k in range(1, 10)),
              f"| total {st[9] - st[0]} cyc" + (f", gap from prev {st[0] - buf[(it - 1) * 16 + 9]}" if it else ""))
    if eng.info["kernel_launches"] > 2:   # tick kernel: per-tick globaltimer (ns) of CTA 0
        rows = sorted((buf[r * 16 + 10], buf[r * 16 + 11], buf[r * 16 + 12]) for r in range(8) if buf[r * 16 + 10])
        for i, (a, b, c) in enumerate(rows):
            gap = f", gap from prev exit {a - rows[i - 1][2]} ns" if i else ""
            print(f"tick: entry->wait-done {b - a} ns, wait-done->exit {c - b} ns{gap}")
        ctas = [(buf[128 + 4 * b], buf[128 + 4 * b + 1], buf[128 + 4 * b + 2]) for b in range(1024)
                if buf[128 + 4 * b]]
        if ctas:
            t0 = min(c[0] for c in ctas)
            ent = sorted(c[0] - t0 for c in ctas)
            wd = sorted(c[1] - t0 for c in ctas)
            ex = sorted(c[2] - t0 for c in ctas)
            work = sorted(c[2] - c[1] for c in ctas)
            print(f"tick 100, {len(ctas)} CTAs (ns from first entry): entry {ent[0]}..{ent[-1]}, "
                  f"wait-done {wd[0]}..{wd[-1]}, exit {ex[0]}..{ex[-1]}, "
                  f"work min/med/max {work[0]}/{work[len(work) // 2]}/{work[-1]}")
    if eng.info["kernel_launches"] == 2:   # resident march: stamps of CTA 0, thread 0 (steps 1-4, last 4)
        rn = ["wait", "load", "compute", "publish", "sync"]
        for r in range(8):
            st = [buf[r * 16 + k] for k in range(6)]
            if st[0] == 0:
                continue
            if st[1] == 0:
                st[1] = st[0]
            d = [st[k] - st[k - 1] for k in range(1, 6)]
            print(f"row {r}: " + " ".join(f"{rn[k]}:{d[k]}" for k in range(5)), f"| total {st[5] - st[0]} cyc")
        g0, g1 = buf[0 * 16 + 6], buf[7 * 16 + 6]
        c0, c1 = buf[0 * 16 + 0], buf[7 * 16 + 0]
        steps = eng.info["steps"] - 1
        print(f"step 1 -> step S: {(g1 - g0) / steps:.1f} ns/step, {(c1 - c0) / steps:.0f} cyc/step, "
              f"clock {(c1 - c0) / max(g1 - g0, 1):.3f} GHz")
