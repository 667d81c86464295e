"""HPG-MxP bench on B200: one JSON line (driver contract).

A "step" is one double-single GMRES-IR solve of the benchmark problem
(27-point stencil, b = A 1, x0 = 0, 4-level V-cycle, restart 30, tol 1e-9,
max 300 iterations -- the reference's timed-phase solve, ref: bench.py:189-213)
at 256^3 rows per GPU (BASELINE.json configs[1]; weak scaling over the
factor_ranks process grid for N > 1).  ``value`` is the HPG-MxP GFLOP/s of the
timed mixed solves, penalised by min(1, n_d / n_ir) from a standard validation
run at the same local size (the reference CLI's headline number,
ref: bench.py:240-270); raw, fp64 and speedup figures ride along.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HPG-MxP GFLOP/s (mixed, and speedup vs fp64) at 1/2/4/8 B200; % HBM roofline"
GS_KERNEL = "k_gs_pass_tma<float,128,8> level-0 colour pass (multicolor GS, fp32; full and zero-guess sweeps)"
UNIT = "GFLOP/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def _env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


# ------------------------------------------------------------------ clocks

class Clocks:
    """nvidia-smi sampling during the timed region (profiling recipe's clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "samples": len(sm),
                "reasons": sorted(reasons)}


# ------------------------------------------------------------------ CPU baseline (oracle)

CPU_L = 64
CPU_ITERS = 10


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_port_sample(iters=CPU_ITERS, L=CPU_L):
    """The oracle port (numpy restatement of the reference) on this host: one mixed
    GMRES-IR solve at L^3 capped at `iters` inner iterations, row loops split over
    every host thread.  Returns (gflops, seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import hpgmxp_oracle as O
    O.set_threads(cpu_threads())
    s = O.Solver(L, L, L, 1, 4)
    b = s.rhs()
    s.count = O.Count()
    t0 = time.perf_counter()
    s.gmres(b, "mixed", 1e-9, iters, 30)
    dt = time.perf_counter() - t0
    return sum(s.count.flops.values()) / dt / 1e9, dt


def run_reference(args):
    rank, world = _env_rank()
    if rank != 0:
        return 0
    for _ in range(args.warmup):
        cpu_port_sample()
    vals, secs = [], []
    for _ in range(args.steps):
        g, dt = cpu_port_sample()
        vals.append(g)
        secs.append(dt)
    v = float(np.mean(vals))
    sample = (f"{CPU_L}^3 local grid (256^3 is infeasible on the host: minutes of setup, hours "
              f"per solve), one mixed GMRES-IR solve capped at {CPU_ITERS} inner iterations per "
              f"step, oracle port (numpy restatement of mxpbench), row loops on {cpu_threads()} "
              "threads, BLAS dots multithreaded")
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(secs)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32",
            "data": "synthetic (the benchmark's own generated 27-point problem)",
            "impl": "reference",
            "config": dict(_config(args.local, args.gpus), reference_sample=f"{CPU_L}^3 on the host"),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cpu_threads(), "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------ our arm

def run_ours(args):
    import torch
    from paper_2507_11512_b200 import _lib
    from paper_2507_11512_b200.bench import BenchConfig, _build_state, _solve, run_validation
    from paper_2507_11512_b200.comm import World, runtime
    from paper_2507_11512_b200.krylov import gmres_solve
    from paper_2507_11512_b200.metrics import MOTIFS, Tally, penalty_factor

    rank, nproc = _env_rank()
    if nproc != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={nproc}")
    rt = runtime()
    world = World(nproc) if nproc > 1 else None
    L = args.local
    cfg = BenchConfig(local_nx=L, local_ny=L, local_nz=L, ranks=nproc, time_seconds=0,
                      max_iters=args.max_iters, validation_mode=args.validation)
    peak, peak_kind = _peaks()

    # validation (n_d, n_ir -> penalty), standard mode on one rank at the local size
    val = None
    if not args.no_validation:
        val = run_validation(cfg, world if world is not None else World(1))

    hier, lv, b = _build_state(cfg, nproc, world, rank)
    ctx = hier.ctx
    n = lv.A_hi.n_rows
    stream = rt.stream

    def barrier():
        torch.cuda.synchronize()
        if world is not None:
            world.barrier()

    def timed(mode, steps, tally=None):
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        l0 = ctx.launches()
        iters = []
        e0.record(stream)
        t0 = time.perf_counter()
        for _ in range(steps):
            res = _solve(cfg, hier, lv, b, world, rank, mode, cfg.tol, cfg.max_iters, tally)
            iters.append(res.iterations)
        e1.record(stream)
        barrier()
        wall = time.perf_counter() - t0
        dev = e0.elapsed_time(e1) / 1e3
        return dev, wall, iters, ctx.launches() - l0, res

    # warm-up
    for _ in range(args.warmup):
        _solve(cfg, hier, lv, b, world, rank, "mixed", cfg.tol, cfg.max_iters)

    def tallied(mode):
        """One tallied solve: model flops/bytes, executed flops, moved bytes (this rank)."""
        t = Tally()
        r = _solve(cfg, hier, lv, b, world, rank, mode, cfg.tol, cfg.max_iters, t)
        return t, r

    # flops of one solve (model, this rank) -- counted on a tallied solve; every
    # timed solve must take the same path (same iteration count)
    tal, res = tallied("mixed")
    flops_rank, xflops_rank = tal.total_flops(), tal.total_exec_flops()
    bytes_rank, moved_rank = tal.total_bytes(), tal.total_moved_bytes()

    clocks = Clocks(rt.device.index)
    clocks.start()
    dev_s, wall_s, iters, launches, last = timed("mixed", args.steps)
    clk = clocks.stop()
    if any(it != res.iterations for it in iters):
        raise RuntimeError(f"timed solves took {iters} iterations, the tallied one {res.iterations}")
    # timing of the dominant motif (GS) inside a timed solve: library CUDA events
    tal2, _ = tallied("mixed")
    gs_bytes, gs_sec = tal2.bytes["GS"], tal2.seconds["GS"]
    l0_bytes, l0_sec, l0_sweeps = tal2.gs_level0_bytes, tal2.gs_level0_seconds, tal2.gs_level0_sweeps
    ncolors = ctx.level_info(0)["ncolors"]
    from paper_2507_11512_b200.multigrid import full_sweep_moved_bytes
    l0_moved = full_sweep_moved_bytes(hier, 4) * l0_sweeps

    # fp64 comparison (same solves in double)
    dtal, dres = tallied("double")
    dflops_rank = dtal.total_flops()
    ddev_s, dwall_s, diters, _, _ = timed("double", args.steps)
    if any(it != dres.iterations for it in diters):
        raise RuntimeError(f"timed fp64 solves took {diters} iterations, the tallied one {dres.iterations}")

    # labelled variants of the mixed solve (same problem, same iteration counts):
    #   general_ell: every row loads its column indices (no implicit-index rows)
    #   lower_sweep: zero-initial-guess sweeps form only the strictly-lower products
    #                (bitwise-identical results, fewer executed flops than counted)
    variants = {}
    for name, opts in (("general_ell", {"stencil": 0}), ("lower_sweep", {"lower": 1})):
        for k, v in opts.items():
            ctx.set_option(k, v)
        _solve(cfg, hier, lv, b, world, rank, "mixed", cfg.tol, cfg.max_iters)  # re-capture graphs
        vt, vr = tallied("mixed")
        vdev, _, viters, _, _ = timed("mixed", args.steps)
        if any(it != vr.iterations for it in viters):
            raise RuntimeError(f"{name}: timed solves took {viters} iterations, the tallied one {vr.iterations}")
        variants[name] = [vdev, vt.total_flops(), vt.total_exec_flops(), vt.total_bytes(), vt.total_moved_bytes()]
        for k in opts:
            ctx.set_option(k, {"stencil": 1, "lower": 0}[k])
    _solve(cfg, hier, lv, b, world, rank, "mixed", cfg.tol, cfg.max_iters)

    # e2e through the public API with host buffers (H2D b, D2H x inside the region)
    # pinned host buffers (the public API accepts numpy arrays; pinned ones DMA directly)
    b_pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
    b_pin.copy_(b)
    b_pin = b_pin.numpy()
    # one zero initial guess per step, prepared before the region (each receives its
    # step's solution in place, as the reference's x0 does)
    x_hosts = [torch.zeros(n, dtype=torch.float64, pin_memory=True).numpy() for _ in range(args.steps)]
    barrier()
    t0 = time.perf_counter()
    for x_host in x_hosts:
        gmres_solve(lv.A_hi, lv.A_lo, hier.preconditioner(), b_pin, x0=x_host, mode="mixed",
                    tol=cfg.tol, max_iters=cfg.max_iters, m=cfg.restart, plan=lv.plan,
                    world=world, rank=rank)
    barrier()
    e2e_s = time.perf_counter() - t0

    # max over ranks, sums of flops over ranks
    def reduce(vals, op):
        if world is None:
            return vals
        parts = world.gather(rank, vals)
        parts = world.broadcast_bytes(parts)
        return [op(p[i] for p in parts) for i in range(len(vals))]

    dev_s, ddev_s, e2e_s, wall_s = reduce([dev_s, ddev_s, e2e_s, wall_s], max)
    flops_all, xflops_all, dflops_all, bytes_all, moved_all = reduce(
        [flops_rank, xflops_rank, dflops_rank, bytes_rank, moved_rank], sum)
    vsum = {}
    for name, (vdev, vf, vx, vb, vm) in variants.items():
        vdev = reduce([vdev], max)[0]
        vf, vx, vb, vm = reduce([vf, vx, vb, vm], sum)
        vsum[name] = (vdev, vf, vx, vb, vm)
    hier.close()
    if rank != 0:
        return 0

    K = args.steps
    raw = flops_all * K / dev_s / 1e9
    penalty = penalty_factor(val["n_d"], val["n_ir"]) if val else None
    value = raw * penalty if penalty is not None else raw
    fp64 = dflops_all * K / ddev_s / 1e9
    gs_gbs = gs_bytes / gs_sec / 1e9 if gs_sec > 0 else 0.0
    l0_gbs = l0_bytes / l0_sec / 1e9 if l0_sec > 0 else 0.0
    l0_launches = l0_sweeps * ncolors
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f)
        if tr.get("local") == L and tr.get("kernel") == GS_KERNEL:
            traffic, traffic_src = tr["gs_pass_level0_f32_dram_bytes_per_launch"], tr["source"]
    except (OSError, KeyError, ValueError):
        pass
    cpu_g, cpu_s = cpu_port_sample() if nproc == 1 and not args.no_cpu else (None, None)
    pk = peak * nproc

    def vline(vdev, vf, vx, vb, vm):
        g = vf * K / vdev / 1e9
        return {"gflops": g * (penalty if penalty is not None else 1.0), "raw_gflops": g,
                "executed_gflops": vx * K / vdev / 1e9, "ms_per_solve": 1e3 * vdev / K,
                "model_bytes_per_solve": vb, "moved_bytes_per_solve": vm,
                "frac_model": vb * K / vdev / 1e9 / pk, "frac_moved": vm * K / vdev / 1e9 / pk}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": nproc, "steps": K,
        "warmup": args.warmup, "ms_per_step": 1e3 * dev_s / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32 (double-single GMRES-IR)",
        "data": "synthetic (the benchmark's own generated 27-point problem, b = A*1)",
        "config": _config(L, nproc),
        "raw_gflops": raw, "penalty": penalty,
        "executed_gflops": xflops_all * K / dev_s / 1e9,
        "flops_note": "value counts the reference's frozen flop model (metrics.py:7-16); the "
                      "headline kernels form every counted product (zero-guess sweeps included, "
                      "as the reference does), so executed_gflops == raw_gflops",
        "validation": val, "iterations_per_solve": iters,
        "fp64_gflops": fp64, "fp64_iterations_per_solve": diters,
        "speedup_vs_fp64": value / fp64 if fp64 else None,
        "solve_roofline": {"model_bytes_per_solve": bytes_all, "moved_bytes_per_solve": moved_all,
                           "achieved_gbs": bytes_all * K / dev_s / 1e9,
                           "achieved_moved_gbs": moved_all * K / dev_s / 1e9,
                           "peak_gbs": pk,
                           "frac": bytes_all * K / dev_s / 1e9 / pk,
                           "frac_moved": moved_all * K / dev_s / 1e9 / pk,
                           "note": "frac: reference byte model (metrics.py:37-77), model-equivalent -- "
                                   "implicit-index rows do not load the 4-B column index it charges; "
                                   "frac_moved: the bytes the kernels move (model minus those indices)"},
        "variants": {
            "general_ell": dict(vline(*vsum["general_ell"]),
                                note="stencil=0: every row loads its int32 column index plane (the "
                                     "paper's general ELL; model bytes == moved bytes)"),
            "lower_sweep": dict(vline(*vsum["lower_sweep"]),
                                note="lower=1: zero-initial-guess sweeps form only the strictly-lower "
                                     "products (bitwise-identical z); gflops counts the model, "
                                     "executed_gflops what ran"),
        },
        "roofline": {"bound": "hbm",
                     "kernel": GS_KERNEL,
                     "achieved": l0_gbs, "peak": peak, "unit": "GB/s",
                     "frac": l0_gbs / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": (l0_bytes / l0_launches) if l0_launches else None,
                     "avg_launch_us": (l0_sec / l0_launches * 1e6) if l0_launches else None,
                     "model_equivalent": True,
                     "moved_bytes_per_launch": (l0_moved / l0_launches) if l0_launches else None,
                     "achieved_moved": l0_moved / l0_sec / 1e9 if l0_sec > 0 else 0.0,
                     "frac_moved": l0_moved / l0_sec / 1e9 / peak if l0_sec > 0 else 0.0,
                     # the DRAM bytes ncu measured for one launch over the live launch time (the
                     # peak is a copy rate; read-dominated streams reach ~7.1 TB/s, so this can pass 1)
                     "frac_dram": (traffic / (l0_sec / l0_launches) / 1e9 / peak)
                     if traffic and l0_sec > 0 and l0_launches else None,
                     "bytes_note": "achieved/frac: SURVEY 8(d) reference model (4-B column index per nonzero), "
                                   "model-equivalent since interior rows compute their columns (implicit-index "
                                   "rows); *_moved: values + indices of face rows + r, z gather, z write",
                     "timing": "library CUDA events around every level-0 sweep of one timed solve",
                     "peak_kind": peak_kind,
                     "gs_all_levels_gbs": gs_gbs},
        # H2D: b and the initial guess x0; D2H: the solution into x0
        "e2e": {"value": value * dev_s / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 2 * n * 8,
                "d2h_bytes_per_step": n * 8},
        "gpu_launches": launches,
        "clocks": clk,
        "wall_seconds": wall_s,
    }
    if cpu_g is not None:
        line["cpu_baseline"] = {
            "value": cpu_g, "unit": UNIT, "cores": cpu_threads(), "kind": "port",
            "sample": f"{CPU_L}^3, one mixed GMRES-IR solve capped at {CPU_ITERS} iterations "
                      f"({cpu_s:.1f} s), oracle numpy port on this host, row loops on "
                      f"{cpu_threads()} threads"}
    print(json.dumps(line))
    return 0


def _config(L, nproc):
    """The workload both arms report (ours measures it; the reference arm times a
    bounded host sample of it and says so)."""
    return {"workload": "HPG-MxP double-single GMRES-IR solve (4-level MG V-cycle, "
                        "multicolor GS, restart 30, tol 1e-9, max 300 it)",
            "local_grid": f"{L}^3 per GPU", "process_grid": list(_grid(nproc)),
            "parallelism": f"3D domain decomposition x{nproc}",
            "l2": "inputs larger than L2 (ELL operands ~7 GB per GPU)"}


def _grid(n):
    from paper_2507_11512_b200.geometry import factor_ranks
    return factor_ranks(n)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--local", type=int, default=256)
    p.add_argument("--max-iters", type=int, default=300)
    p.add_argument("--no-validation", action="store_true")
    p.add_argument("--validation", choices=("standard", "fullscale"), default="standard",
                   help="standard: 1-rank solve at the local size; fullscale: all ranks, full problem")
    p.add_argument("--no-cpu", action="store_true")
    args = p.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
