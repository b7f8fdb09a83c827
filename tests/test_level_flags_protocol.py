"""CPU model of the resident level march's flag protocol (csrc/ridc_levels.cuh),
the device-side form of the reference's LevelBuffer watermark / released
protocol (engine.py:284-331).

Each level runs in its own thread exactly the per-step sequence of the
kernel's thread 0 (one segment): acquire-wait for the producer's published
step (cached), read the window slots, release the slots below the next
window, publish deferred and batched (every K steps, and always before a
backpressure wait), wait for the consumer's release before a slot is
reused, store the new step at the start of the next step.  Random delays
shuffle the interleavings; inbox rings are at the kernel's minimum
(levels + 2).  Every window read must find exactly the producer step it
asks for (no overwrite, no stale slot) and the pipeline must finish (no
deadlock) -- the same properties the GPU tests check bitwise on one device
(tests/test_gpu_reslevels.py::test_resident_levels_tight_inboxes) and the
multi-GPU ranks rely on."""

import random
import threading
import time

import pytest


class Flag:
    def __init__(self):
        self.v = 0
        self.cv = threading.Condition()

    def store(self, v):
        with self.cv:
            self.v = v
            self.cv.notify_all()

    def wait_geq(self, want, timeout=10.0):
        with self.cv:
            ok = self.cv.wait_for(lambda: self.v >= want, timeout)
        if not ok:
            raise TimeoutError(f"flag stuck at {self.v} < {want}")
        return self.v


def run_model(levels, per, cap, pub_every, seed, epochs=2, backpressure=True, slow_consumers=1.0):
    rng = random.Random(seed)
    delays = [[rng.random() * 2e-4 * (slow_consumers if j > 0 else 1.0) for _ in range(per + 2)]
              for j in range(levels)]
    for epoch in range(1, epochs + 1):          # flag values carry the run epoch
        ep = epoch << 32
        inbox = [[None] * cap for _ in range(levels)]      # inbox[j]: level j-1's states
        pub = [Flag() for _ in range(levels)]              # pub[j]: in level j's memory
        rel = [Flag() for _ in range(levels)]              # rel[j]: level j's released-below
        for j in range(1, levels):
            inbox[j][0] = (epoch, 0)                       # seeded step 0
        errors = []

        def level(j):
            try:
                out = j < levels - 1
                seen_in = seen_rel = 0
                published = 0
                pend = 0

                def store(ts):
                    inbox[j + 1][ts % cap] = (epoch, ts)

                for t in range(1, per + 1):
                    steady = t >= j
                    if j > 0:
                        need = ep | (t if steady else j)
                        if seen_in < need:
                            seen_in = pub[j].wait_geq(need)
                    if pend:
                        store(pend)                        # step t-1 to the consumer
                    if j > 0:
                        for a in range(j + 1):
                            s = t - a if steady else a
                            got = inbox[j][s % cap]
                            if got != (epoch, s):
                                raise AssertionError(f"level {j} step {t}: slot of step {s} holds {got}")
                    time.sleep(delays[j][t])               # the solve
                    if out and t > 1 and (t - 1) % pub_every == 0:
                        pub[j + 1].store(ep | (t - 1))
                        published = t - 1
                    if j > 0:
                        rel[j].store(ep | max(0, t + 1 - j))
                    if out:
                        need_rel = t - cap + 1
                        if backpressure and need_rel > 0 and seen_rel < (ep | need_rel):
                            if published < t - 1:
                                pub[j + 1].store(ep | (t - 1))
                                published = t - 1
                            seen_rel = rel[j + 1].wait_geq(ep | need_rel)
                        pend = t
                if out and pend:
                    store(pend)
                    pub[j + 1].store(ep | pend)
            except Exception as exc:                       # surfaced below
                errors.append(exc)
                for f in pub + rel:                        # unblock the others
                    f.store(1 << 62)

        th = [threading.Thread(target=level, args=(j,)) for j in range(levels)]
        for x in th:
            x.start()
        for x in th:
            x.join(30)
        assert not any(x.is_alive() for x in th), "pipeline deadlocked"
        if errors:
            raise errors[0]


@pytest.mark.parametrize("levels", [2, 3, 4, 8])
@pytest.mark.parametrize("pub_every", [1, 4, 7])
def test_flag_protocol_minimum_rings(levels, pub_every):
    run_model(levels, per=levels * (levels + 1) // 2 + 40, cap=levels + 2, pub_every=pub_every, seed=levels * 10 + pub_every)


def test_flag_protocol_default_pipe_rings():
    # the memop protocol's minimum inbox, 2j+5 slots (here j = 1; the ranks' default is 2j+13)
    run_model(4, per=60, cap=7, pub_every=4, seed=7)


def test_model_detects_a_missing_backpressure_wait():
    """The model is not vacuous: a producer that never waits for its
    consumer's release overwrites window slots still being read."""
    with pytest.raises(AssertionError):
        run_model(3, per=60, cap=5, pub_every=1, seed=3, epochs=1, backpressure=False, slow_consumers=20.0)
