"""CPU level rank for the distributed-protocol tests (gloo, no GPU).

TEST INFRASTRUCTURE: one RIDC level per process, stepping with the CPU
oracle (oracle/ridc_oracle.c) and exchanging each published slot
(state, f^S, f^N) point to point with torch.distributed send/recv -- the
reference's LevelBuffer.publish / claim_rows (engine.py:305-328) across
processes.  It plugs into the product's interval driver
(paper_1209_4297_b200.distributed.run_levels), so the re-seed / interval
protocol the GPU ranks use is exercised with world_size > 1 on CPU.
"""

import numpy as np
import torch
import torch.distributed as dist

from oracle import oracle as O
from paper_1209_4297_b200.quadrature import startup_weights, steady_weights


class OracleLevel:
    def __init__(self, pd, levels, steps, restarts, dt, rank, world):
        self.pd, self.L, self.per, self.dt = pd, levels, steps // restarts, dt
        self.j, self.world = rank, world
        self.n = pd.nx * pd.ny

    def _send(self, arrs):
        dist.send(torch.from_numpy(np.concatenate(arrs)), dst=self.j + 1)

    def _recv(self):
        buf = torch.empty(3 * self.n, dtype=torch.float64)
        dist.recv(buf, src=self.j - 1)
        a = buf.numpy()
        return a[:self.n].copy(), a[self.n:2 * self.n].copy(), a[2 * self.n:].copy()

    def run_interval(self, r, state0):
        j, pd, dt, per = self.j, self.pd, self.dt, self.per
        state0 = np.asarray(state0, dtype=np.float64)
        fs0, fn0 = O.stiff(pd, state0), O.nonstiff(pd, state0)
        hist = {0: (fs0, fn0)}          # previous level's published slots (step -> (fs, fn))
        eta = state0.copy()
        for t in range(1, per + 1):
            if j == 0:
                eta, fs, fn = O.predict_step(pd, dt, eta)
            else:
                hi = j if t < j else t                     # _window_span, engine.py:124-128
                while max(hist) < hi:
                    _s, fsr, fnr = self._recv()
                    hist[max(hist) + 1] = (fsr, fnr)
                if t < j:                                  # startup: oldest first
                    idx = list(range(0, j + 1))
                    i_new, i_old = t, t - 1
                    w = startup_weights(j, t - 1, dt).weights
                else:                                      # steady: newest first
                    idx = list(range(t, t - j - 1, -1))
                    i_new, i_old = 0, 1
                    w = steady_weights(j, dt).weights
                fs_win = np.array([hist[s][0] for s in idx])
                fn_win = np.array([hist[s][1] for s in idx])
                eta, fs, fn = O.correct_step(pd, dt, eta, fs_win, fn_win, i_new, i_old, w)
                for s in [s for s in hist if s < t + 1 - j]:   # release_through
                    if s != max(hist):
                        del hist[s]
            if j < self.world - 1:
                self._send([eta, fs, fn])
        return eta, 0.0


def gloo_broadcast(world):
    def bcast(x, is_top):
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).clone()
        dist.broadcast(t, src=world - 1)
        return t.numpy()
    return bcast
