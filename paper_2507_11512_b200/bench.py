"""Benchmark orchestration and CLI, device edition (ref: bench.py:1-377).

Three phases, as in the reference: validation (fp64 GMRES vs GMRES-IR ->
n_d, n_ir), the timed mixed-precision phase (repeat until the time budget is
spent, at least once) and the same number of fp64 solves.  Each rank is one
process on one GPU (launch with ``torchrun --nproc-per-node N`` for N > 1);
the report has the reference's schema plus additive keys (wall seconds,
model bytes, roofline fraction, device).
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from dataclasses import asdict, dataclass

import numpy as np

from .comm import ProtocolError, TopologyError, World, reduce_sum
from .geometry import CoarseningError, GlobalProblem
from .krylov import gmres_solve
from .metrics import MOTIFS, Tally, emit_report, gflops, penalty_factor, sum_motif_dicts
from .multigrid import build_hierarchy
from .problem import generate_rhs
from .smoother import SmootherWorkspace


class ConfigError(Exception):
    """The benchmark configuration is invalid (ref: bench.py:36-37)."""


class ValidationError(Exception):
    """The fp64 reference solve did not converge (ref: bench.py:40-41)."""


VALIDATION_MODES = ("standard", "fullscale")
COLORING_STRATEGIES = ("greedy", "jpl")


@dataclass
class BenchConfig:
    """Every knob of a run; defaults are the reference's desk settings (ref: bench.py:48-104)."""

    local_nx: int = 16
    local_ny: int = 16
    local_nz: int = 16
    ranks: int = 1
    restart: int = 30
    tol: float = 1e-9
    max_iters: int = 300
    nd_cap: int = 10000
    time_seconds: float = 5.0
    validation_mode: str = "standard"
    validation_ranks: int = 1
    coloring: str = "greedy"
    seed: int = 0
    mg_levels: int = 4
    nu1: int = 1
    nu2: int = 1
    nu_c: int = 1
    # (npx, npy, npz) for the job's ranks instead of factor_ranks(ranks) -- an
    # extension of the reference, used to run x-axis splits on 2 and 4 GPUs
    proc_grid: tuple = None

    def validate(self):
        if self.mg_levels < 1:
            raise ConfigError("mg_levels must be at least 1")
        q = 1 << (self.mg_levels - 1)
        for name in ("local_nx", "local_ny", "local_nz"):
            d = getattr(self, name)
            if d < 1:
                raise ConfigError(f"{name} = {d} must be positive")
            if d % q:
                raise ConfigError(f"{name} = {d} is not divisible by {q} "
                                  f"(needed for {self.mg_levels} grid levels)")
        checks = [
            (self.ranks >= 1, "ranks must be at least 1"),
            (1 <= self.validation_ranks <= self.ranks, "validation_ranks must lie in [1, ranks]"),
            (self.restart >= 1, "restart length must be at least 1"),
            (self.tol > 0, "tol must be positive"),
            (self.max_iters >= 1 and self.nd_cap >= 1, "iteration caps must be at least 1"),
            (self.time_seconds >= 0, "time_seconds must be non-negative"),
            (self.validation_mode in VALIDATION_MODES,
             f"unknown validation mode {self.validation_mode!r}"),
            (self.coloring in COLORING_STRATEGIES, f"unknown coloring strategy {self.coloring!r}"),
            (min(self.nu1, self.nu2, self.nu_c) >= 1, "smoothing sweep counts must be at least 1"),
            (self.proc_grid is None or (len(self.proc_grid) == 3 and min(self.proc_grid) >= 1 and
                                        int(np.prod(self.proc_grid)) == self.ranks),
             f"process grid {self.proc_grid} does not hold {self.ranks} ranks"),
        ]
        for ok, msg in checks:
            if not ok:
                raise ConfigError(msg)

    def sweeps(self):
        return SmootherWorkspace(nu1=self.nu1, nu2=self.nu2, nu_c=self.nu_c)


# -- per-rank state -------------------------------------------------------------

def _build_state(cfg, nranks, world, rank):
    dims = cfg.proc_grid if (cfg.proc_grid is not None and nranks == cfg.ranks) else None
    gp = GlobalProblem.from_local(cfg.local_nx, cfg.local_ny, cfg.local_nz, nranks, proc_dims=dims)
    hier = build_hierarchy(gp.domain(rank), cfg.mg_levels, world, rank,
                           strategy=cfg.coloring, seed=cfg.seed, sweeps=cfg.sweeps())
    lv = hier.levels[0]
    return hier, lv, generate_rhs(lv.A_hi).b


def _solve(cfg, hier, lv, b, world, rank, mode, tol, max_iters, tally=None, x0=None):
    """Zero initial guess, V-cycle preconditioner (ref: bench.py:123-133)."""
    import torch
    if x0 is None:
        x0 = torch.zeros(lv.A_hi.n_rows, dtype=torch.float64, device=b.device)
    return gmres_solve(lv.A_hi, lv.A_lo, hier.preconditioner(tally), b, x0=x0, mode=mode,
                       tol=tol, max_iters=max_iters, m=cfg.restart, plan=lv.plan,
                       world=world, rank=rank, tally=tally)


# -- phase 1 --------------------------------------------------------------------

def _validation_worker(world, rank, cfg, nranks):
    hier, lv, b = _build_state(cfg, nranks, world, rank)
    try:
        dres = _solve(cfg, hier, lv, b, world, rank, "double", cfg.tol, cfg.nd_cap)
        if cfg.validation_mode == "standard":
            if not dres.converged:
                raise ValidationError(f"double GMRES did not reach {cfg.tol:g} within "
                                      f"{cfg.nd_cap} iterations (relres {dres.relres:.3e})")
            target = cfg.tol
        else:
            target = cfg.tol if dres.converged else dres.relres
        mres = _solve(cfg, hier, lv, b, world, rank, "mixed", target, cfg.nd_cap)
    finally:
        hier.close()
    return dres.iterations, mres.iterations, dres.relres, mres.relres


def run_validation(cfg, world=None):
    """n_d and n_ir on the validation problem (ref: bench.py:157-183)."""
    cfg.validate()
    here = world if world is not None else _job_world(cfg)
    if cfg.validation_mode == "standard":
        nranks = cfg.validation_ranks
    else:
        nranks = cfg.ranks
    if nranks > here.nranks:
        raise ConfigError(f"validation on {nranks} ranks but the job has {here.nranks}")
    if nranks == 1:
        out = None
        if here.rank == 0:
            out = _validation_worker(None, 0, cfg, 1)
        out = here.broadcast_bytes(out)
    elif nranks == here.nranks:
        out = here.run(_validation_worker, cfg, nranks)[0]
    else:
        # the first `nranks` processes form the validation world (factor_ranks grid
        # of nranks, ref: bench.py:165-167); the others wait for its result
        sub = here.subworld(nranks)
        out = sub.run(_validation_worker, cfg, nranks)[0] if sub is not None else None
        out = here.broadcast_bytes(out)
    n_d, n_ir, res_d, _ = out
    return {"mode": cfg.validation_mode, "n_d": n_d, "n_ir": n_ir, "ratio": n_d / n_ir,
            "residual": res_d}


# -- phases 2 and 3 ---------------------------------------------------------------

def _bench_worker(world, rank, cfg):
    import torch
    hier, lv, b = _build_state(cfg, cfg.ranks, world, rank)
    tally_mxp, tally_dbl = Tally(), Tally()
    iters_mxp, iters_dbl = [], []
    wall_mxp = wall_dbl = 0.0
    try:
        t0 = time.perf_counter()
        reps = 0
        while True:
            ts = time.perf_counter()
            res = _solve(cfg, hier, lv, b, world, rank, "mixed", cfg.tol, cfg.max_iters, tally_mxp)
            torch.cuda.current_stream().synchronize()
            wall_mxp += time.perf_counter() - ts
            iters_mxp.append(res.iterations)
            reps += 1
            flag = 1.0 if rank == 0 and time.perf_counter() - t0 < cfg.time_seconds else 0.0
            if reduce_sum(world, rank, flag) == 0.0:
                break
        for _ in range(reps):
            ts = time.perf_counter()
            res = _solve(cfg, hier, lv, b, world, rank, "double", cfg.tol, cfg.max_iters, tally_dbl)
            torch.cuda.current_stream().synchronize()
            wall_dbl += time.perf_counter() - ts
            iters_dbl.append(res.iterations)
    finally:
        hier.close()
    return {"reps": reps, "iters_mxp": iters_mxp, "iters_dbl": iters_dbl,
            "mxp": {"flops": dict(tally_mxp.flops), "bytes": dict(tally_mxp.bytes),
                    "seconds": dict(tally_mxp.seconds), "wall_seconds": wall_mxp},
            "double": {"flops": dict(tally_dbl.flops), "bytes": dict(tally_dbl.bytes),
                       "seconds": dict(tally_dbl.seconds), "wall_seconds": wall_dbl}}


def _phase_block(parts, phase):
    """Flops summed over ranks, rank-0 seconds (ref: bench.py:226-237)."""
    flops = sum_motif_dicts([p[phase]["flops"] for p in parts])
    seconds = parts[0][phase]["seconds"]
    return {m: {"seconds": seconds[m], "flops": flops[m],
                "gflops": gflops(flops[m], seconds[m]) if seconds[m] > 0 else 0.0}
            for m in MOTIFS}


def _assemble_report(cfg, val, parts, peak_gbs=None):
    mxp = _phase_block(parts, "mxp")
    dbl = _phase_block(parts, "double")
    penalty = penalty_factor(val["n_d"], val["n_ir"])
    tot_f = sum(mxp[m]["flops"] for m in MOTIFS)
    tot_s = sum(mxp[m]["seconds"] for m in MOTIFS)
    raw = gflops(tot_f, tot_s) if tot_s > 0 else 0.0
    dbl_f = sum(dbl[m]["flops"] for m in MOTIFS)
    dbl_s = sum(dbl[m]["seconds"] for m in MOTIFS)
    dbl_total = gflops(dbl_f, dbl_s) if dbl_s > 0 else 0.0
    motif_speedup = {m: (mxp[m]["gflops"] * penalty / dbl[m]["gflops"]
                         if dbl[m]["gflops"] > 0 else 0.0) for m in MOTIFS}
    summary = {"raw_gflops": raw, "penalty": penalty, "penalized_gflops": raw * penalty,
               "speedup": raw * penalty / dbl_total if dbl_total > 0 else 0.0,
               "motif_speedup": motif_speedup, "reps": parts[0]["reps"]}
    # additive keys (not in the reference schema)
    wall = parts[0]["mxp"]["wall_seconds"]
    mbytes = sum(sum(p["mxp"]["bytes"].values()) for p in parts)
    summary["wall_seconds"] = wall
    summary["wall_gflops"] = gflops(tot_f, wall) if wall > 0 else 0.0
    summary["hbm_bytes_model"] = mbytes
    if peak_gbs and wall > 0:
        summary["roofline_fraction"] = mbytes / wall / 1e9 / (peak_gbs * len(parts))
    return {"config": asdict(cfg), "validation": val, "mxp": mxp, "double": dbl,
            "summary": summary}


def _job_world(cfg):
    nproc = int(os.environ.get("WORLD_SIZE", "1"))
    if cfg.ranks != nproc:
        raise ProtocolError(f"{cfg.ranks} ranks requested but {nproc} process(es) running; "
                            f"launch with torchrun --nproc-per-node {cfg.ranks}")
    return World(nproc)


def run_benchmark(cfg):
    """All three phases; returns the report dict on every rank (ref: bench.py:273-282)."""
    cfg.validate()
    world = _job_world(cfg)
    val = run_validation(cfg, world)
    parts = world.run(_bench_worker, cfg)
    peak = None
    try:
        import json
        with open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "MEASURED_PEAKS.json")) as f:
            peak = json.load(f).get("hbm_gbs")
    except OSError:
        pass
    return _assemble_report(cfg, val, parts, peak)


def dump_matrix(cfg, path):
    """Rank 0's local block in MatrixMarket form, natural order, global ids (ref: bench.py:288-295)."""
    from .problem import host_level
    gp = GlobalProblem.from_local(cfg.local_nx, cfg.local_ny, cfg.local_nz, cfg.ranks)
    dom = gp.domain(0)
    vals, cols, nnz, diag, meta = host_level(dom.local_dims, dom.coords, dom.proc_dims)
    from .coloring import greedy_coloring
    col = greedy_coloring(*dom.local_dims)
    lx, ly, _ = dom.local_dims
    # permuted row -> global row / column ids
    nat = col.perm
    x, y, z = nat % lx, (nat // lx) % ly, nat // (lx * ly)
    grow = (dom.ox + x) + dom.gnx * ((dom.oy + y) + dom.gny * (dom.oz + z))
    order = np.argsort(nat)  # rows in natural order
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{gp.n_global} {gp.n_global} {int(nnz.sum())}\n")
        for i in order:
            gi = int(grow[i])
            xi, yi, zi = x[i], y[i], z[i]
            for s in range(int(nnz[i])):
                # recover the neighbour's global id from the stencil offset order
                f.write(f"{gi + 1} {int(_neighbour_gid(dom, xi, yi, zi, s, nnz[i])) + 1} "
                        f"{_fmt(vals[i, s])}\n")


def _neighbour_gid(dom, x, y, z, slot, nnz):
    s = 0
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                gx, gy, gz = dom.ox + x + dx, dom.oy + y + dy, dom.oz + z + dz
                if 0 <= gx < dom.gnx and 0 <= gy < dom.gny and 0 <= gz < dom.gnz:
                    if s == slot:
                        return gx + dom.gnx * (gy + dom.gny * gz)
                    s += 1
    raise IndexError(slot)


def _fmt(v):
    return str(int(v)) if float(v).is_integer() else repr(float(v))


# -- CLI ----------------------------------------------------------------------------

def _build_parser():
    p = argparse.ArgumentParser(prog="mxpbench", description=(
        "Mixed-precision multigrid GMRES benchmark on a 27-point stencil problem "
        "(B200 device solver)."))
    p.add_argument("--local-nx", type=int, default=16)
    p.add_argument("--local-ny", type=int, default=16)
    p.add_argument("--local-nz", type=int, default=16)
    p.add_argument("--ranks", type=int, default=None,
                   help="ranks = processes = GPUs (default: WORLD_SIZE or 1)")
    p.add_argument("--restart", type=int, default=30)
    p.add_argument("--tol", type=float, default=1e-9)
    p.add_argument("--max-iters", type=int, default=300)
    p.add_argument("--time-seconds", type=float, default=5.0)
    p.add_argument("--validation", choices=VALIDATION_MODES, default="standard")
    p.add_argument("--coloring", choices=COLORING_STRATEGIES, default="greedy")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--report-path", default=None, metavar="PATH")
    p.add_argument("--dump-matrix", default=None, metavar="PATH")
    return p


def main(argv=None):
    args = _build_parser().parse_args(argv)
    ranks = args.ranks if args.ranks is not None else int(os.environ.get("WORLD_SIZE", "1"))
    cfg = BenchConfig(local_nx=args.local_nx, local_ny=args.local_ny, local_nz=args.local_nz,
                      ranks=ranks, restart=args.restart, tol=args.tol,
                      max_iters=args.max_iters, time_seconds=args.time_seconds,
                      validation_mode=args.validation, coloring=args.coloring, seed=args.seed)
    try:
        cfg.validate()
        if args.dump_matrix and int(os.environ.get("RANK", "0")) == 0:
            dump_matrix(cfg, args.dump_matrix)
        report = run_benchmark(cfg)
    except (ConfigError, CoarseningError) as exc:
        print(f"configuration error: {exc}", file=sys.stderr)
        return 2
    except ValidationError as exc:
        print(f"validation failed: {exc}", file=sys.stderr)
        return 3
    except (ProtocolError, TopologyError) as exc:
        print(f"protocol error: {exc}", file=sys.stderr)
        return 4
    except NotImplementedError as exc:
        print(f"configuration error: {exc}", file=sys.stderr)
        return 2
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    text = emit_report(report)
    if args.report_path:
        with open(args.report_path, "w") as fh:
            fh.write(text + "\n")
        s = report["summary"]
        print(f"penalized {s['penalized_gflops']:.3f} GFLOP/s (penalty {s['penalty']:.3f}, "
              f"speedup {s['speedup']:.2f}x); report written to {args.report_path}")
    else:
        print(text)
    return 0


def console_main():
    sys.exit(main())


if __name__ == "__main__":
    console_main()
