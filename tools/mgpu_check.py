"""Multi-GPU parity driver (launched by tests/test_multigpu.py under torchrun).

Every rank builds its box of a decomposed problem, runs SpMV / GS / V-cycle on
random data and compares bitwise with the CPU oracle's all-rank simulation, then
runs the fp64 and mixed solves and compares iteration counts with the reference
fixtures.  Rank 0 prints one JSON line with the verdicts."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    levels = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    # optional explicit process grid "px,py,pz" (x-axis splits on 2 / 4 GPUs)
    dims = tuple(int(v) for v in sys.argv[3].split(",")) if len(sys.argv) > 3 else None
    import torch
    import hpgmxp_oracle as O
    from paper_2507_11512_b200.comm import World
    from paper_2507_11512_b200.geometry import GlobalProblem
    from paper_2507_11512_b200.krylov import gmres_solve, spmv
    from paper_2507_11512_b200.multigrid import build_hierarchy
    from paper_2507_11512_b200.problem import generate_rhs
    from paper_2507_11512_b200.smoother import forward_gs_sweep

    world = World()
    rank, R = world.rank, world.nranks
    gp = GlobalProblem.from_local(L, L, L, R, proc_dims=dims)
    h = build_hierarchy(gp.domain(rank), levels, world, rank)
    lv = h.levels[0]
    A, Alo = lv.A_hi, lv.A_lo
    n, ne = A.n_rows, A.n_cols_extended
    ora = O.Solver(L, L, L, R, levels, dims=dims)
    ok = {}
    # structure
    OL = ora.L(0)[rank]
    ok["structure"] = bool(np.array_equal(A.col_idx, OL.col_idx) and np.array_equal(A.values, OL.values))
    rng = [np.random.default_rng(100 + q) for q in range(R)]
    for dt, tdt, Ad in ((np.float64, torch.float64, A), (np.float32, torch.float32, Alo)):
        xs = [g.standard_normal(ora.L(0)[q].n).astype(dt) for q, g in enumerate(rng)]
        rs = [g.standard_normal(ora.L(0)[q].n).astype(dt) for q, g in enumerate(rng)]
        xe = []
        for q in range(R):
            v = np.zeros(ora.L(0)[q].n_ext, dtype=dt)
            v[:len(xs[q])] = xs[q]
            xe.append(v)
        yo = ora.spmv([v.copy() for v in xe])
        xd = torch.zeros(ne, dtype=tdt, device="cuda")
        xd[:n] = torch.from_numpy(xs[rank]).cuda()
        yd = spmv(Ad, xd).cpu().numpy()
        ok[f"spmv_{np.dtype(dt).name}"] = bool(np.array_equal(yd, yo[rank]))
        zo = [v.copy() for v in xe]
        ora.gs_sweep(0, rs, zo, z_is_zero=False)
        zd = torch.zeros(ne, dtype=tdt, device="cuda")
        zd[:n] = torch.from_numpy(xs[rank]).cuda()
        forward_gs_sweep(Ad, torch.from_numpy(rs[rank]).cuda(), zd)
        ok[f"gs_{np.dtype(dt).name}"] = bool(np.array_equal(zd[:n].cpu().numpy(), zo[rank][:n]))
        vo = ora.vcycle([r.copy() for r in rs])
        vd = h.apply(torch.from_numpy(rs[rank]).cuda()).cpu().numpy()
        ok[f"vcycle_{np.dtype(dt).name}"] = bool(np.array_equal(vd, vo[rank]))
    b = generate_rhs(A).b
    res = {}
    for mode in ("double", "mixed"):
        x0 = torch.zeros(n, dtype=torch.float64, device="cuda")
        r = gmres_solve(A, Alo, h.preconditioner(), b, x0=x0, mode=mode, tol=1e-9, max_iters=300,
                        m=30, plan=lv.plan, world=world, rank=rank, debug_replication=True)
        res[mode] = {"iterations": r.iterations, "relres": r.relres, "converged": r.converged,
                     "cycles": r.cycle_iterations,
                     "x_err": float((x0 - 1.0).abs().max().item())}
    h.close()
    # the reference's full pipeline on the same world: fullscale validation (all
    # ranks) + timed phases; builds two more hierarchies (fresh NCCL communicators)
    from paper_2507_11512_b200.bench import BenchConfig, run_benchmark
    rep = run_benchmark(BenchConfig(local_nx=L, local_ny=L, local_nz=L, ranks=R, time_seconds=0,
                                    mg_levels=levels, validation_mode="fullscale", proc_grid=dims))
    allok = world.gather(rank, ok)
    if rank == 0:
        print(json.dumps({"ranks": R, "local": L, "proc_dims": list(gp.domain(0).proc_dims),
                          "checks": allok, "solves": res,
                          "validation": rep["validation"], "summary": rep["summary"]}))


if __name__ == "__main__":
    main()
