"""Per-component CUDA-event timings at L^3 (warm, repeated).  Not a bench number:
used to tune kernels between bench runs.  Prints one JSON dict."""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--local", type=int, default=256)
    p.add_argument("--reps", type=int, default=20)
    p.add_argument("--cgs", default="", help="label: time CGS2 for every k of a restart cycle and exit")
    p.add_argument("--brief", default="", help="label: print only the headline keys on one line")
    a = p.parse_args()
    import torch
    from paper_2507_11512_b200 import _lib
    from paper_2507_11512_b200.bench import BenchConfig, _build_state, _solve
    from paper_2507_11512_b200.krylov import GmresWorkspace
    cfg = BenchConfig(local_nx=a.local, local_ny=a.local, local_nz=a.local, time_seconds=0)
    hier, lv, b = _build_state(cfg, 1, None, 0)
    ctx = hier.ctx
    st = ctx.stream
    n, ne = lv.A_hi.n_rows, lv.A_hi.n_cols_extended
    nnz = lv.A_hi.nnz_total
    out = {"local": a.local, "tail_rows": os.environ.get("HPG_TAIL_ROWS", "default"),
           "zero_sweep_slots_per_row": ctx.level_info(0)["zero_sweep_slots"] / n,
           "stencil_rows_L0": ctx.level_info(0)["stencil_rows"] if os.environ.get("HPG_STENCIL", "1") != "0" else 0}

    def timeit(fn, reps=a.reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3  # us

    if a.cgs:
        ws = GmresWorkspace.allocate(n, 30, np.float32, device="cuda")
        ws.Q.normal_()
        w = torch.randn(n, device="cuda", dtype=torch.float32)
        res = np.zeros(64)
        ts = []
        for k in range(30):
            ts.append(timeit(lambda: ctx.call("hpg_cgs2", _lib.F32, _lib.ptr(ws.Q), ws.Q.stride(0), k, _lib.ptr(w),
                                              _lib.ptr(ws.Q[k + 1]), res.ctypes.data_as(C.POINTER(C.c_double))),
                             reps=5))
        byts = [(3 * n * (k + 1) * 4 + 7 * n * 4) for k in range(30)]
        print(a.cgs, "total_us", round(sum(ts), 1), "eff", round(sum(byts) / sum(ts) / 1e3 / 6553.9, 3),
              [round(t) for t in ts])
        hier.close()
        return
    x32 = torch.randn(ne, device="cuda", dtype=torch.float32)
    y32 = torch.empty(n, device="cuda", dtype=torch.float32)
    r32 = torch.randn(n, device="cuda", dtype=torch.float32)
    z32 = torch.zeros(ne, device="cuda", dtype=torch.float32)
    us = timeit(lambda: ctx.call("hpg_spmv", 0, _lib.F32, _lib.ptr(x32), _lib.ptr(y32)))
    out["spmv_f32_us"] = us
    out["spmv_f32_GBs"] = (nnz * 8 + 2 * n * 4) / us / 1e3
    x64 = torch.randn(ne, device="cuda", dtype=torch.float64)
    r64 = torch.empty(n, device="cuda", dtype=torch.float64)
    b64 = torch.randn(n, device="cuda", dtype=torch.float64)
    rho = C.c_double()
    us = timeit(lambda: ctx.call("hpg_residual", _lib.ptr(b64), _lib.ptr(x64), _lib.ptr(r64), C.byref(rho)))
    out["residual_f64_us"] = us
    out["residual_f64_GBs"] = (nnz * 12 + 3 * n * 8) / us / 1e3
    us = timeit(lambda: ctx.call("hpg_gs_sweep", 0, _lib.F32, _lib.ptr(r32), _lib.ptr(z32), 0))
    out["gs_sweep_L0_f32_us"] = us
    out["gs_sweep_L0_f32_GBs"] = (nnz * 8 + 3 * n * 4) / us / 1e3
    out["gs_sweep0_L0_f32_us"] = timeit(lambda: ctx.call("hpg_gs_sweep", 0, _lib.F32, _lib.ptr(r32), _lib.ptr(z32), 1))
    z64 = torch.zeros(ne, device="cuda", dtype=torch.float64)
    r64b = torch.randn(n, device="cuda", dtype=torch.float64)
    us = timeit(lambda: ctx.call("hpg_gs_sweep", 0, _lib.F64, _lib.ptr(r64b), _lib.ptr(z64), 0))
    out["gs_sweep_L0_f64_us"] = us
    out["gs_sweep_L0_f64_GBs"] = (nnz * 12 + 3 * n * 8) / us / 1e3
    y64 = torch.empty(n, device="cuda", dtype=torch.float64)
    us = timeit(lambda: ctx.call("hpg_spmv", 0, _lib.F64, _lib.ptr(x64), _lib.ptr(y64)))
    out["spmv_f64_us"] = us
    out["spmv_f64_GBs"] = (nnz * 12 + 2 * n * 8) / us / 1e3
    # every level's sweeps, restriction and prolongation (fp32), warm
    for li in range(1, len(hier.levels)):
        A = hier.levels[li].A_lo
        nl, nel = A.n_rows, A.n_cols_extended
        rl = torch.randn(nl, device="cuda", dtype=torch.float32)
        zl = torch.zeros(nel, device="cuda", dtype=torch.float32)
        out[f"gs_sweep_L{li}_f32_us"] = timeit(
            lambda: ctx.call("hpg_gs_sweep", li, _lib.F32, _lib.ptr(rl), _lib.ptr(zl), 0))
        out[f"gs_sweep0_L{li}_f32_us"] = timeit(
            lambda: ctx.call("hpg_gs_sweep", li, _lib.F32, _lib.ptr(rl), _lib.ptr(zl), 1))
    for li in range(len(hier.levels) - 1):
        Af, Ac = hier.levels[li].A_lo, hier.levels[li + 1].A_lo
        rf = torch.randn(Af.n_rows, device="cuda", dtype=torch.float32)
        zf = torch.randn(Af.n_cols_extended, device="cuda", dtype=torch.float32)
        rc = torch.empty(Ac.n_rows, device="cuda", dtype=torch.float32)
        zc = torch.randn(Ac.n_cols_extended, device="cuda", dtype=torch.float32)
        out[f"restrict_L{li}_f32_us"] = timeit(
            lambda: ctx.call("hpg_restrict", li, _lib.F32, _lib.ptr(rf), _lib.ptr(zf), _lib.ptr(rc)))
        out[f"prolong_L{li}_f32_us"] = timeit(
            lambda: ctx.call("hpg_prolong", li, _lib.F32, _lib.ptr(zf), _lib.ptr(zc)))
    us = timeit(lambda: hier.apply(r32, out=z32))
    out["vcycle_f32_us"] = us
    us = timeit(lambda: hier.apply(r64 if False else b64, out=x64))
    out["vcycle_f64_us"] = us
    # model bytes of one V-cycle (f32)
    from paper_2507_11512_b200.metrics import Tally
    from paper_2507_11512_b200.multigrid import count_vcycle
    t = Tally()
    count_vcycle(hier, t, np.float32)
    out["vcycle_f32_model_GBs"] = t.total_bytes() / out["vcycle_f32_us"] / 1e3
    ws = GmresWorkspace.allocate(n, 30, np.float32, device="cuda")
    ws.Q.normal_()
    w = torch.randn(n, device="cuda", dtype=torch.float32)
    res = np.zeros(64)
    for k in (0, 7, 15, 29):
        us = timeit(lambda: ctx.call("hpg_cgs2", _lib.F32, _lib.ptr(ws.Q), ws.Q.stride(0), k, _lib.ptr(w),
                                     _lib.ptr(ws.Q[k + 1]), res.ctypes.data_as(C.POINTER(C.c_double))), reps=5)
        kb = k + 1
        out[f"cgs2_k{kb}_us"] = us
        out[f"cgs2_k{kb}_modelGBs"] = (4 * n * kb * 4 + 4 * n * 4 + 3 * n * 4) / us / 1e3
    # one restart cycle of the real solve
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _solve(cfg, hier, lv, b, None, 0, "mixed", 1e-9, 30)
    tal = Tally()
    e0.record(st)
    res_ = _solve(cfg, hier, lv, b, None, 0, "mixed", 1e-9, 30, tal)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out["solve30_ms"] = ms
    out["solve30_model_GBs"] = tal.total_bytes() / ms / 1e6
    out["solve30_GFs"] = tal.total_flops() / ms / 1e6
    out["solve30_motif_s"] = tal.seconds
    if a.brief:
        keys = ("gs_sweep_L0_f32_us", "gs_sweep0_L0_f32_us", "zero_sweep_slots_per_row", "gs_sweep_L0_f64_us", "vcycle_f32_us", "vcycle_f64_us", "spmv_f32_us",
                "cgs2_k30_us", "solve30_ms", "spmv_f64_us", "residual_f64_us", "restrict_L0_f32_us", "stencil_rows_L0", "gs_sweep_L1_f32_us", "gs_sweep0_L1_f32_us", "gs_sweep_L2_f32_us",
                "gs_sweep0_L2_f32_us", "gs_sweep_L3_f32_us", "gs_sweep0_L3_f32_us")
        print(a.brief, {k: round(v, 1) for k, v in out.items() if k in keys})
    else:
        print(json.dumps(out))
    hier.close()


if __name__ == "__main__":
    main()
