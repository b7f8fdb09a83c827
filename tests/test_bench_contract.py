"""bench.py's reference arm runs on the CPU (the oracle port) and prints one
JSON line with the driver's contract keys; under torchrun the non-zero ranks
exit without output (the bench contract)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=300, env=e, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    return r.stdout.strip()


def test_reference_arm_contract():
    out = _run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--sample-steps", "4"])
    lines = [ln for ln in out.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "c2-reaction-diffusion-1d" and d["config"]["points"] == 1 << 20
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["dtype"] == "f64" and d["vs_baseline"] is None


def test_reference_arm_nonzero_rank_is_silent():
    out = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0"],
               env={"RANK": "1", "WORLD_SIZE": "2"})
    assert out == ""


def test_workloads_keep_the_configuration_dt():
    """--nt shortens the horizon, never changes dt (explicit terms of the 2-D kinds)."""
    sys.path.insert(0, ROOT)
    import bench
    for name, dt in (("c2", 1e-4), ("c3", 0.02 / 1000), ("c4", 0.05 / 1000)):
        for nt in (None, 20):
            sysm, n_t, cfg = bench.workload(name, 4096 if name != "c2" else None, nt)
            ivp = sysm.ivp
            assert abs((ivp.t_end - ivp.t_start) / n_t - dt) <= 1e-15, (name, nt)
            assert cfg["nt"] == n_t
