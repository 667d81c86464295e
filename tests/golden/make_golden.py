"""Generate the golden fixtures in tests/golden/ from the REFERENCE package.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``mxpbench`` from /root/reference/pkg/src read-only and writes
compressed .npz / .json fixtures next to this script.  The fixtures travel
with the repo; nothing at test time reads /root/reference.

Solve fixtures are produced twice, with OPENBLAS_NUM_THREADS=1 and with the
default thread count, because the reference's dot products go through
OpenBLAS and mixed-precision iteration counts depend on the reduction order
(SURVEY.md 0.8).  The pair gives the envelope the GPU solver is judged against.
"""

import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"


def _import_ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import mxpbench  # noqa: F401
    return mxpbench


def _problem(lx, ly, lz, ranks, dims=None):
    """The reference's GlobalProblem; ``dims`` = an explicit (npx, npy, npz) grid
    (the reference's frozen dataclass built directly -- its from_local always
    factors, which never splits x below 8 ranks)."""
    from mxpbench.geometry import GlobalProblem
    if dims is None:
        return GlobalProblem.from_local(lx, ly, lz, ranks)
    px, py, pz = dims
    assert px * py * pz == ranks
    return GlobalProblem(nx=px * lx, ny=py * ly, nz=pz * lz, npx=px, npy=py, npz=pz,
                         lnx=lx, lny=ly, lnz=lz)


# ---------------------------------------------------------------------------
# structure: ELL arrays, permutation, halo plans, injection maps
# ---------------------------------------------------------------------------

STRUCT_CASES = {
    # name: (lx, ly, lz, ranks, levels)
    "s468": (4, 6, 8, 1, 2),
    "s16": (16, 16, 16, 1, 4),
    "s8": (8, 8, 8, 1, 4),
    "odd354": (3, 5, 4, 1, 1),
    "odd7": (7, 7, 7, 1, 1),
    "deg144": (1, 4, 4, 1, 1),
    "deg414": (4, 1, 4, 1, 1),
    "deg114": (1, 1, 4, 1, 1),
    "deg111": (1, 1, 1, 1, 1),
    "r2": (4, 4, 4, 2, 2),
    "r4": (4, 4, 4, 4, 2),
    "r8": (4, 4, 4, 8, 2),
    "r8x8": (8, 8, 8, 8, 4),
    "r3": (4, 4, 4, 3, 1),
    "r12": (4, 4, 2, 12, 1),
}

# explicit process grids that split x (x faces, xy / xz edges, corners below 8 ranks)
XSPLIT_STRUCT = {
    # name: (lx, ly, lz, ranks, levels, dims)
    "x211": (4, 4, 4, 2, 2, (2, 1, 1)),
    "x221": (4, 4, 4, 4, 2, (2, 2, 1)),
    "x212": (4, 4, 4, 4, 2, (2, 1, 2)),
    "x411": (4, 4, 4, 4, 1, (4, 1, 1)),
}
XSPLIT_KERNELS = {"kx211": (8, 2, 3, (2, 1, 1)), "kx221": (8, 4, 3, (2, 2, 1)), "kx212": (8, 4, 3, (2, 1, 2))}
XSPLIT_SOLVES = [
    # name, local, ranks, levels, m, max_iters, dims
    ("x211l16", 16, 2, 4, 30, 300, (2, 1, 1)),
    ("x221l8", 8, 4, 4, 30, 300, (2, 2, 1)),
    ("x212l8", 8, 4, 4, 30, 300, (2, 1, 2)),
]


def _level_arrays(prefix, lv, out):
    A = lv.A_hi
    out[prefix + "values"] = A.values
    out[prefix + "col_idx"] = A.col_idx
    out[prefix + "row_nnz"] = A.row_nnz
    out[prefix + "diag_pos"] = A.diag_pos
    out[prefix + "perm"] = lv.coloring.perm
    out[prefix + "color"] = lv.coloring.color
    out[prefix + "color_offsets"] = lv.coloring.color_offsets
    out[prefix + "n_ext"] = np.array(A.n_cols_extended)
    if lv.f2c is not None:
        out[prefix + "f2c"] = lv.f2c
    plan = lv.plan
    out[prefix + "neighbors"] = np.array(plan.neighbors, dtype=np.int64)
    for nb in plan.neighbors:
        out[prefix + f"send_{nb}"] = plan.send_rows[nb]
        sl = plan.recv_slices[nb]
        out[prefix + f"recv_{nb}"] = np.array([sl.start, sl.stop])


def make_structure(xsplit=False):
    mx = _import_ref()
    from mxpbench.comm import RankWorld
    from mxpbench.geometry import GlobalProblem
    from mxpbench.multigrid import build_hierarchy

    cases = {k: v + (None,) for k, v in STRUCT_CASES.items()} if not xsplit else XSPLIT_STRUCT
    for name, (lx, ly, lz, ranks, levels, dims) in cases.items():
        gp = _problem(lx, ly, lz, ranks, dims)
        out = {"dims": np.array([lx, ly, lz, ranks, levels])}
        if dims is not None:
            out["proc_dims"] = np.array(dims)

        def worker(world, rank):
            return build_hierarchy(gp.domain(rank), levels, world, rank)

        if ranks == 1:
            hiers = [worker(None, 0)]
        else:
            hiers = RankWorld(ranks).run(worker)
        for r, h in enumerate(hiers):
            for li, lv in enumerate(h.levels):
                _level_arrays(f"r{r}_l{li}_", lv, out)
        np.savez_compressed(os.path.join(HERE, f"struct_{name}.npz"), **out)
        print("struct", name)
    del mx


# ---------------------------------------------------------------------------
# kernels on random data (single rank 16^3, and 8 ranks of 4^3)
# ---------------------------------------------------------------------------

def make_kernels(xsplit=False):
    _import_ref()
    from mxpbench.comm import RankWorld, exchange
    from mxpbench.geometry import GlobalProblem
    from mxpbench.krylov import spmv
    from mxpbench.multigrid import build_hierarchy, fused_residual_restrict, prolong_add
    from mxpbench.smoother import forward_gs_sweep

    def run_rank(world, rank, gp, levels, seed):
        h = build_hierarchy(gp.domain(rank), levels, world, rank)
        rng = np.random.default_rng(seed + rank)
        out = {}
        for dt, tag in ((np.float64, "f64"), (np.float32, "f32")):
            lv = h.levels[0]
            A = lv.A_hi if dt == np.float64 else lv.A_lo
            n, ne = A.n_rows, A.n_cols_extended
            x = np.zeros(ne, dtype=dt)
            x[:n] = rng.standard_normal(n).astype(dt)
            r = rng.standard_normal(n).astype(dt)
            out[f"{tag}_x"] = x[:n].copy()
            out[f"{tag}_r"] = r.copy()
            out[f"{tag}_spmv"] = spmv(A, x.copy(), lv.plan, world, rank)
            z = np.zeros(ne, dtype=dt)
            forward_gs_sweep(A, r, z, lv.coloring, lv.plan, world, rank, z_is_zero=True)
            out[f"{tag}_gs0"] = z[:n].copy()
            z2 = x.copy()
            forward_gs_sweep(A, r, z2, lv.coloring, lv.plan, world, rank)
            out[f"{tag}_gs1"] = z2[:n].copy()
            # restriction of r - A x at injected rows (fresh halo)
            x3 = x.copy()
            exchange(x3, lv.plan, world, rank)
            nxt = h.levels[1]
            out[f"{tag}_restrict"] = fused_residual_restrict(A, r, x3, nxt.f2c).copy()
            xc = rng.standard_normal(nxt.A_hi.n_rows).astype(dt)
            out[f"{tag}_xc"] = xc
            xf = x.copy()
            prolong_add(xf, xc, nxt.f2c)
            out[f"{tag}_prolong"] = xf[:n].copy()
            out[f"{tag}_vcycle"] = h.apply(r.copy()).copy()
        return out

    cases = {"k16": (16, 1, 4, None), "k8r8": (4, 8, 2, None), "k8x8r8": (8, 8, 4, None),
             "k8r2": (8, 2, 3, None)} if not xsplit else XSPLIT_KERNELS
    for name, (l, ranks, levels, dims) in cases.items():
        gp = _problem(l, l, l, ranks, dims)
        if ranks == 1:
            parts = [run_rank(None, 0, gp, levels, 7)]
        else:
            parts = RankWorld(ranks).run(run_rank, gp, levels, 7)
        out = {"dims": np.array([l, l, l, ranks, levels])}
        if dims is not None:
            out["proc_dims"] = np.array(dims)
        for r, p in enumerate(parts):
            for k, v in p.items():
                out[f"r{r}_{k}"] = v
        np.savez_compressed(os.path.join(HERE, f"kernels_{name}.npz"), **out)
        print("kernels", name)


# ---------------------------------------------------------------------------
# solves (child process per OpenBLAS thread setting)
# ---------------------------------------------------------------------------

SOLVE_CASES = [
    # name, local, ranks, levels, m, max_iters, modes
    ("l16", 16, 1, 4, 30, 300),
    ("l32", 32, 1, 4, 30, 300),
    ("l4m5", 4, 1, 3, 5, 300),
    ("r8l8", 8, 8, 4, 30, 300),
    ("r2l16", 16, 2, 4, 30, 300),
]


def _solve_child(case):
    _import_ref()
    import mxpbench.krylov as kry
    from mxpbench.comm import RankWorld
    from mxpbench.geometry import GlobalProblem
    from mxpbench.multigrid import build_hierarchy

    name, l, ranks, levels, m, max_iters = case[:6]
    gp = _problem(l, l, l, ranks, case[6] if len(case) > 6 else None)
    result = {}
    orig = kry.givens_update
    for mode in ("double", "mixed"):
        ks = {}

        def logged(H, t, c, s, k, _ks=ks):
            import threading
            _ks.setdefault(threading.current_thread().name, []).append(k)
            return orig(H, t, c, s, k)

        kry.givens_update = logged

        def worker(world, rank):
            h = build_hierarchy(gp.domain(rank), levels, world, rank)
            lv = h.levels[0]
            b = lv.A_hi.values.sum(axis=1)
            x0 = np.zeros(lv.A_hi.n_rows)
            res = kry.gmres_solve(lv.A_hi, lv.A_lo, lambda r: h.apply(r), b, x0=x0,
                                  mode=mode, tol=1e-9, max_iters=max_iters, m=m,
                                  plan=lv.plan, world=world, rank=rank)
            return res, x0

        if ranks == 1:
            outs = [worker(None, 0)]
        else:
            outs = RankWorld(ranks).run(worker)
        kry.givens_update = orig
        res = outs[0][0]
        klist = ks.get("rank-0") or next(iter(ks.values()))
        cycles, cur = [], 0
        for k in klist:
            if k == 0 and cur:
                cycles.append(cur)
                cur = 0
            cur += 1
        if cur:
            cycles.append(cur)
        result[mode] = {"iterations": res.iterations, "restarts": res.restarts,
                        "relres": res.relres, "converged": res.converged,
                        "cycle_iters": cycles,
                        "pairs": [list(map(float, p)) for p in res.boundary_pairs]}
        xs = np.concatenate([o[1] for o in outs])
        result[mode]["_x"] = xs
    return result


def make_solves(xsplit=False):
    out = {}
    cases = XSPLIT_SOLVES if xsplit else SOLVE_CASES
    for threads in ("1", "default"):
        env = dict(os.environ)
        env["PYTHONDONTWRITEBYTECODE"] = "1"
        if threads == "1":
            env["OPENBLAS_NUM_THREADS"] = "1"
        else:
            env.pop("OPENBLAS_NUM_THREADS", None)
        for case in cases:
            cmd = [sys.executable, __file__, "--solve-child", json.dumps(case)]
            p = subprocess.run(cmd, env=env, capture_output=True, text=True, check=True)
            out.setdefault(case[0], {})[threads] = json.loads(p.stdout.strip().splitlines()[-1])
            print("solve", case[0], threads, {k: v["iterations"] for k, v in
                                             out[case[0]][threads].items()})
    xs = {}
    for name, d in out.items():
        for threads, modes in d.items():
            for mode, r in modes.items():
                path = r.pop("_xpath")
                xs[f"{name}_{threads}_{mode}"] = np.load(path)
                os.unlink(path)
    tag = "_xsplit" if xsplit else ""
    np.savez_compressed(os.path.join(HERE, f"solves{tag}_x.npz"), **xs)
    with open(os.path.join(HERE, f"solves{tag}.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


def make_jpl():
    """JPL colorings (ref: coloring.py:56-70) and a JPL hierarchy's V-cycle/solve."""
    _import_ref()
    from mxpbench.geometry import GlobalProblem
    from mxpbench.multigrid import build_hierarchy
    from mxpbench.problem import generate_matrix
    from mxpbench.coloring import color
    out = {}
    for (lx, ly, lz, seed) in [(4, 4, 4, 0), (6, 4, 8, 3), (8, 8, 8, 11), (5, 3, 4, 7), (16, 16, 16, 0)]:
        A = generate_matrix(GlobalProblem.from_local(lx, ly, lz, 1).domain(0))
        c = color(A, "jpl", seed=seed)
        key = f"{lx}x{ly}x{lz}_s{seed}"
        out[f"color_{key}"] = c.color
        out[f"perm_{key}"] = c.perm
        out[f"offsets_{key}"] = c.color_offsets
    # 16^3, 4 levels, jpl seed 0: level arrays, f2c, a V-cycle on random data
    h = build_hierarchy(GlobalProblem.from_local(16, 16, 16, 1).domain(0), 4, strategy="jpl", seed=0)
    rng = np.random.default_rng(5)
    for li, lv in enumerate(h.levels):
        out[f"h_l{li}_col_idx"] = lv.A_hi.col_idx
        out[f"h_l{li}_perm"] = lv.coloring.perm
        out[f"h_l{li}_offsets"] = lv.coloring.color_offsets
        if lv.f2c is not None:
            out[f"h_l{li}_f2c"] = lv.f2c
    for dt, tag in ((np.float64, "f64"), (np.float32, "f32")):
        r = rng.standard_normal(h.levels[0].A_hi.n_rows).astype(dt)
        out[f"h_r_{tag}"] = r
        out[f"h_vcycle_{tag}"] = h.apply(r.copy()).copy()
    from mxpbench.krylov import gmres_solve
    lv = h.levels[0]
    b = lv.A_hi.values.sum(axis=1)
    for mode in ("double", "mixed"):
        res = gmres_solve(lv.A_hi, lv.A_lo, lambda v: h.apply(v), b, x0=np.zeros(lv.A_hi.n_rows),
                          mode=mode, tol=1e-9, max_iters=300, m=30)
        out[f"h_solve_{mode}"] = np.array([res.iterations, res.relres])
    np.savez_compressed(os.path.join(HERE, "jpl.npz"), **out)
    print("jpl")


def make_validation():
    _import_ref()
    from mxpbench.bench import BenchConfig, run_validation
    out = {}
    for name, cfg in {
        "std16": BenchConfig(),
        "std4l3": BenchConfig(local_nx=4, local_ny=4, local_nz=4, mg_levels=3),
        "full8r8": BenchConfig(local_nx=8, local_ny=8, local_nz=8, ranks=8,
                               validation_mode="fullscale"),
    }.items():
        out[name] = run_validation(cfg)
        print("validation", name, out[name])
    with open(os.path.join(HERE, "validation.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--solve-child":
        case = json.loads(sys.argv[2])
        res = _solve_child(case)
        import tempfile
        for mode, r in res.items():
            fd, path = tempfile.mkstemp(suffix=".npy")
            os.close(fd)
            np.save(path, r.pop("_x"))
            r["_xpath"] = path
        print(json.dumps(res))
        sys.exit(0)
    what = sys.argv[1:] or ["structure", "kernels", "solves", "validation", "jpl"]
    if "structure" in what:
        make_structure()
    if "kernels" in what:
        make_kernels()
    if "solves" in what:
        make_solves()
    if "validation" in what:
        make_validation()
    if "jpl" in what:
        make_jpl()
    if "xsplit" in what:  # explicit x-splitting process grids (written to separate files)
        make_structure(xsplit=True)
        make_kernels(xsplit=True)
        make_solves(xsplit=True)
    if "xsplit-kernels" in what:
        make_kernels(xsplit=True)
# MatrixMarket fixtures (tests/golden/mtx_sha256.json) were produced with:
#   from mxpbench.bench import BenchConfig, dump_matrix
#   dump_matrix(BenchConfig(local_nx=8, local_ny=8, local_nz=8), path)              -> "l8r1"
#   dump_matrix(BenchConfig(local_nx=4, ..., ranks=2, mg_levels=2), path)            -> "l4r2"
#   dump_matrix(BenchConfig(local_nx=4, ..., ranks=8, mg_levels=2), path)            -> "l4r8"
# and hashed with hashlib.sha256 over the file bytes.
