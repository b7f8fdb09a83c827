"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py           # golden.npz + cases.json
    python tests/golden/make_golden.py --paper   # golden_paper.npz + cases_paper.json

It imports the reference package read-only (PYTHONPATH=/root/reference/pkg/src),
runs ``ridc.engine.run_serial`` / ``run_pipelined`` and single steps under
``threadpool_limits(1)`` (as studies.py:265 does), and writes
``tests/golden/golden.npz`` plus ``tests/golden/cases.json`` (inputs and
configurations).  Tests on the GPU box only read these committed files.

For the problem kinds the reference does not ship (1-D/2-D reaction-diffusion,
2-D advection-diffusion) the script builds the equivalent reference
``SplitIVP`` from dense operators at small n, so the reference itself stays
the oracle there.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from threadpoolctl import threadpool_limits  # noqa: E402

from ridc import engine as R  # noqa: E402
from ridc import ivp as RI  # noqa: E402
from ridc import kernels as RK  # noqa: E402
from ridc import problems as RP  # noqa: E402
from ridc import quadrature as RQ  # noqa: E402
from ridc import steppers as RS  # noqa: E402

from paper_1209_4297_b200 import problems as P  # noqa: E402


def _periodic_second_diff(n, coef):
    m = np.zeros((n, n))
    for i in range(n):
        m[i, i] = -2.0 * coef
        m[i, (i - 1) % n] = coef
        m[i, (i + 1) % n] = coef
    return m


def ref_ivp(pd, y0, t_end):
    """Reference SplitIVP equivalent to a descriptor (dense operators, small n)."""
    n = pd.nx * pd.ny
    if pd.kind == P.KIND_REACTION_DIFFUSION_1D:
        dif = _periodic_second_diff(pd.nx, pd.d_x / pd.h_x ** 2)
        rho = pd.rho
        return RI.SplitIVP(n, 0.0, t_end, y0, eval_nonstiff=lambda t, u: rho * u * (1.0 - u),
                           eval_stiff=lambda t, u: RK.mat_vec(dif, u), stiff_linear_operator=dif)
    if pd.kind in (P.KIND_ADV_DIFF_2D, P.KIND_REACTION_DIFFUSION_2D):
        nx, ny = pd.nx, pd.ny
        dxx = np.kron(np.eye(ny), _periodic_second_diff(nx, pd.d_x / pd.h_x ** 2))
        cdy = pd.d_y / pd.h_y ** 2
        fnm = np.zeros((n, n))
        for r in range(ny):
            for c in range(nx):
                i = r * nx + c
                up = ((r + 1) % ny) * nx + c
                dn = ((r - 1) % ny) * nx + c
                fnm[i, i] += -2.0 * cdy
                fnm[i, up] += cdy
                fnm[i, dn] += cdy
                if pd.kind == P.KIND_ADV_DIFF_2D:
                    cax, cay = pd.c_x / pd.h_x, pd.c_y / pd.h_y
                    fnm[i, i] += -cax - cay
                    fnm[i, r * nx + (c + 1) % nx] += cax
                    fnm[i, up] += cay
        if pd.kind == P.KIND_ADV_DIFF_2D:
            fn = lambda t, u: RK.mat_vec(fnm, u)  # noqa: E731
        else:
            rho = pd.rho
            fn = lambda t, u: rho * u * (1.0 - u) + RK.mat_vec(fnm, u)  # noqa: E731
        return RI.SplitIVP(n, 0.0, t_end, y0, eval_nonstiff=fn,
                           eval_stiff=lambda t, u: RK.mat_vec(dxx, u), stiff_linear_operator=dxx)
    raise ValueError(pd.kind)


def desc_dict(pd):
    return {k: getattr(pd, k) for k in ("kind", "nx", "ny", "c_x", "c_y", "d_x", "d_y", "rho", "h_x", "h_y")}


def main():
    arrays = {}
    cases = []

    def add_run(name, pd, y0, ivp, t_end, levels, steps, restarts=1, traj=False, workers=1):
        cfg = R.RidcConfig(levels=levels, steps=steps, restarts=restarts, workers=workers,
                           record_trajectory=traj)
        runner = R.run_pipelined if workers > 1 else R.run_serial
        sol = runner(ivp, cfg)
        arrays[f"{name}/y0"] = np.asarray(y0)
        arrays[f"{name}/final"] = sol.final_state
        arrays[f"{name}/level_finals"] = np.array(sol.level_finals)
        if traj:
            arrays[f"{name}/trajectory"] = sol.trajectory
        cases.append({"name": name, "problem": desc_dict(pd), "t_end": t_end, "levels": levels,
                      "steps": steps, "restarts": restarts, "trajectory": traj,
                      "workers": workers, "ref_wall_seconds": sol.wall_seconds})
        print(f"{name}: wall {sol.wall_seconds:.2f}s  |final|={np.abs(sol.final_state).max():.6g}")

    with threadpool_limits(1):
        # --- reference problems via the reference's own builders -------------
        for (name, dx, t_end, levels, steps, restarts, traj) in [
            ("ad_n128_p1", 1 / 128, 0.5, 1, 50, 1, True),
            ("ad_n128_p4_r2", 1 / 128, 0.5, 4, 60, 2, True),
            ("ad_n200_p3", 1 / 200, 4.0, 3, 100, 1, False),
            ("ad_c1_p1", 1 / 1024, 4.0, 1, 1000, 1, False),
            ("ad_c1_p2", 1 / 1024, 4.0, 2, 1000, 1, False),
            ("ad_c1_p4", 1 / 1024, 4.0, 4, 1000, 1, False),
            ("ad_c1_p4_r10", 1 / 1024, 4.0, 4, 1000, 10, False),
            ("ad_c1_p8", 1 / 1024, 4.0, 8, 1000, 1, False),
        ]:
            spec = RP.AdvectionDiffusionSpec(dx=dx, t_end=t_end)
            sysr = RP.build_advection_diffusion(spec)
            ours = P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=dx, t_end=t_end))
            add_run(name, ours.problem, sysr.ivp.initial_state, sysr.ivp, t_end, levels, steps,
                    restarts, traj)
        for (name, dx, t_end, levels, steps, restarts) in [
            ("bu_n255_p4", 1 / 256, 0.5, 4, 500, 1),
            ("bu_c1_p4", 1 / 1024, 1.0, 4, 1000, 1),
            ("bu_c1_p1", 1 / 1024, 1.0, 1, 1000, 1),
        ]:
            spec = RP.BurgersSpec(dx=dx, t_end=t_end)
            sysr = RP.build_burgers(spec)
            ours = P.build_burgers(P.BurgersSpec(dx=dx, t_end=t_end))
            add_run(name, ours.problem, sysr.ivp.initial_state, sysr.ivp, t_end, levels, steps, restarts)
        # non-finite detection: the same Burgers grid with a CFL-violating dt blows up;
        # the reference raises NonFiniteStateError naming (level, step)
        try:
            sysb = RP.build_burgers(RP.BurgersSpec(dx=1 / 256, t_end=0.5))
            R.run_serial(sysb.ivp, R.RidcConfig(levels=1, steps=100))
            raise SystemExit("expected a blow-up")
        except Exception as exc:  # NonFiniteStateError
            cases.append({"name": "bu_n255_blowup", "problem": desc_dict(P.build_burgers(
                P.BurgersSpec(dx=1 / 256, t_end=0.5)).problem), "t_end": 0.5, "levels": 1,
                "steps": 100, "restarts": 1, "error": type(exc).__name__, "message": str(exc)})
            print("blowup:", exc)
        # the reference's own determinism gate: pipelined (4 workers) == serial, bitwise
        spec = RP.AdvectionDiffusionSpec(dx=1 / 128, t_end=0.5)
        sysr = RP.build_advection_diffusion(spec)
        add_run("ad_n128_p4_pipelined_w4", P.build_advection_diffusion(
            P.AdvectionDiffusionSpec(dx=1 / 128, t_end=0.5)).problem,
            sysr.ivp.initial_state, sysr.ivp, 0.5, 4, 60, 2, False, workers=4)

        # --- new kinds through equivalent reference SplitIVPs ------------------
        rd = P.build_reaction_diffusion(P.ReactionDiffusionSpec(d=1e-3, n=256, t_end=0.5))
        for levels in (1, 2, 4):
            add_run(f"rd_n256_p{levels}", rd.problem, rd.ivp.initial_state,
                    ref_ivp(rd.problem, rd.ivp.initial_state, 0.5), 0.5, levels, 80)
        # stiff variant (r ~ 100): exercises the solve far from identity
        rds = P.build_reaction_diffusion(P.ReactionDiffusionSpec(d=2e-2, n=512, t_end=0.4))
        add_run("rd_n512_stiff_p3", rds.problem, rds.ivp.initial_state,
                ref_ivp(rds.problem, rds.ivp.initial_state, 0.4), 0.4, 3, 40)
        ad2 = P.build_advection_diffusion_2d(P.AdvectionDiffusion2DSpec(nx=32, ny=24, t_end=0.05,
                                                                         dxx=2e-2, dyy=1e-3))
        add_run("ad2d_32x24_p4", ad2.problem, ad2.ivp.initial_state,
                ref_ivp(ad2.problem, ad2.ivp.initial_state, 0.05), 0.05, 4, 40)
        rd2 = P.build_reaction_diffusion_2d(P.ReactionDiffusion2DSpec(nx=32, ny=32, t_end=0.1,
                                                                      dxx=1e-2, dyy=1e-3))
        add_run("rd2d_32x32_p3", rd2.problem, rd2.ivp.initial_state,
                ref_ivp(rd2.problem, rd2.ivp.initial_state, 0.1), 0.1, 3, 30)

        # --- ARK comparators (steppers.integrate_ark with the imex3 / imex4 pairs) --
        from ridc import tableaus as RT

        def add_ark(name, pd, ivp, y0, t_end, scheme, steps):
            tab = RT.imex3_tableau() if scheme == "imex3" else RT.imex4_tableau()
            solver = RS.ImplicitSolver()
            final = RS.integrate_ark(ivp, tab, 0.0, np.array(y0), t_end, steps, solver)
            arrays[f"ark/{name}/y0"] = np.asarray(y0)
            arrays[f"ark/{name}/final"] = final
            cases.append({"name": f"ark/{name}", "problem": desc_dict(pd), "t_end": t_end,
                          "scheme": scheme, "steps": steps})
            print(f"ark/{name}: |final|={np.abs(final).max():.6g}")

        for scheme in ("imex3", "imex4"):
            sysr = RP.build_advection_diffusion(RP.AdvectionDiffusionSpec(dx=1 / 128, t_end=0.5))
            ours = P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 128, t_end=0.5))
            add_ark(f"ad_n128_{scheme}", ours.problem, sysr.ivp, sysr.ivp.initial_state, 0.5, scheme, 40)
            sysb = RP.build_burgers(RP.BurgersSpec(dx=1 / 256, t_end=0.5))
            oursb = P.build_burgers(P.BurgersSpec(dx=1 / 256, t_end=0.5))
            add_ark(f"bu_n255_{scheme}", oursb.problem, sysb.ivp, sysb.ivp.initial_state, 0.5, scheme, 500)
        sysr = RP.build_advection_diffusion(RP.AdvectionDiffusionSpec(dx=1 / 1024, t_end=4.0))
        ours = P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 1024, t_end=4.0))
        add_ark("ad_c1_imex4", ours.problem, sysr.ivp, sysr.ivp.initial_state, 4.0, "imex4", 200)
        rda = P.build_reaction_diffusion(P.ReactionDiffusionSpec(d=2e-2, n=512, t_end=0.4))
        add_ark("rd_n512_stiff_imex3", rda.problem, ref_ivp(rda.problem, rda.ivp.initial_state, 0.4),
                rda.ivp.initial_state, 0.4, "imex3", 40)
        ad2a = P.build_advection_diffusion_2d(P.AdvectionDiffusion2DSpec(nx=32, ny=24, t_end=0.05,
                                                                          dxx=2e-2, dyy=1e-3))
        add_ark("ad2d_32x24_imex4", ad2a.problem, ref_ivp(ad2a.problem, ad2a.ivp.initial_state, 0.05),
                ad2a.ivp.initial_state, 0.05, "imex4", 40)

        # --- single-step KATs ---------------------------------------------------
        solver = RS.ImplicitSolver()
        sc = RI.scalar_ivp(0.0, 1.0, 1.0, stiff_coeff=-1.0)
        y1 = RS.fbe_step(sc, 0.0, np.array([1.0]), 0.5, solver)
        arrays["kat/fbe_scalar"] = y1            # SPEC.md:173 -> 2/3
        spec = RP.AdvectionDiffusionSpec(dx=1 / 64, t_end=1.0)
        sysr = RP.build_advection_diffusion(spec)
        dt = 0.01
        solver.prepare(sysr.ivp.stiff_linear_operator, [dt])
        eta = sysr.ivp.initial_state.copy()
        e1, fs1, fn1 = R.predict_step(sysr.ivp, 0.0, eta, dt, solver)
        arrays["kat/predict/eta_new"], arrays["kat/predict/fs"], arrays["kat/predict/fn"] = e1, fs1, fn1
        # a level-2 steady correction from a synthetic previous-level window
        rng = np.random.default_rng(7)
        win_states = [eta + 0.01 * rng.standard_normal(eta.shape) for _ in range(3)]
        fs_w = np.array([RK.mat_vec(sysr.diffusion_matrix, s) for s in win_states])
        fn_w = np.array([RK.mat_vec(sysr.advection_matrix, s) for s in win_states])
        w = RQ.steady_weights(2, dt)
        ec, fsc, fnc = R.correct_step(2, sysr.ivp, 0.0, eta,
                                      R.LevelWindow(fs_w, fn_w, 0, 1), w, dt, solver)
        arrays["kat/correct/window_states"] = np.array(win_states)
        arrays["kat/correct/eta_new"], arrays["kat/correct/fs"], arrays["kat/correct/fn"] = ec, fsc, fnc
        arrays["kat/correct/fs_win"], arrays["kat/correct/fn_win"] = fs_w, fn_w
        cases.append({"name": "kat/predict", "problem": desc_dict(
            P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 64, t_end=1.0)).problem),
            "dt": dt})
        # Burgers flux KAT: (1,2,3) interior -> -2/dx
        arrays["kat/burgers_flux"] = RK.burgers_flux(np.array([1.0, 2.0, 3.0]), 1.0 / (4 * 0.1))
        arrays["kat/startup_delay"] = np.array([R.startup_delay(j) for j in range(8)])

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(cases, f, indent=1)
    print("wrote", len(arrays), "arrays")


def paper_runs():
    """The paper's own run (adv-diff c=0.1, d=1e-3,
    dx=1e-3, T=40, 4000 steps, RIDC4 with 1 and 10 restarts) and C1 at the
    paper horizon (dx=1/1024, T=40, 1000 steps: r ~ 42), through the
    reference's own run_serial.  Written to golden_paper.npz / cases_paper.json
    (kept apart from golden.npz so that re-running one set leaves the other
    untouched)."""
    arrays = {}
    cases = []
    with threadpool_limits(1):
        for (name, dx, t_end, levels, steps, restarts) in [
            ("paper_p4_r1", 1e-3, 40.0, 4, 4000, 1),
            ("paper_p4_r10", 1e-3, 40.0, 4, 4000, 10),
            ("ad_c1_T40_p1", 1 / 1024, 40.0, 1, 1000, 1),
            ("ad_c1_T40_p4", 1 / 1024, 40.0, 4, 1000, 1),
            # the engine's maximum order (12 levels, engine.py:47) on the C1 grid
            ("ad_c1_p12", 1 / 1024, 0.4, 12, 200, 1),
        ]:
            spec = RP.AdvectionDiffusionSpec(dx=dx, t_end=t_end)
            sysr = RP.build_advection_diffusion(spec)
            ours = P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=dx, t_end=t_end))
            sol = R.run_serial(sysr.ivp, R.RidcConfig(levels=levels, steps=steps, restarts=restarts))
            arrays[f"{name}/y0"] = np.asarray(sysr.ivp.initial_state)
            arrays[f"{name}/final"] = sol.final_state
            arrays[f"{name}/level_finals"] = np.array(sol.level_finals)
            cases.append({"name": name, "problem": desc_dict(ours.problem), "t_end": t_end, "levels": levels,
                          "steps": steps, "restarts": restarts, "trajectory": False, "workers": 1,
                          "ref_wall_seconds": sol.wall_seconds})
            print(f"{name}: wall {sol.wall_seconds:.2f}s  |final|={np.abs(sol.final_state).max():.6g}", flush=True)
    np.savez_compressed(os.path.join(HERE, "golden_paper.npz"), **arrays)
    with open(os.path.join(HERE, "cases_paper.json"), "w") as f:
        json.dump(cases, f, indent=1)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    if "--paper" in sys.argv:
        paper_runs()
    else:
        main()
