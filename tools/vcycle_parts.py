"""Per-level pieces of a V-cycle at L^3 (CUDA events, warm, repeated): forward
sweeps (zero-guess and full), restriction and prolongation at every level, the
whole V-cycle, SpMV and a CGS2 step.  Not a bench number; tells where a V-cycle's
time goes.

    python tools/vcycle_parts.py [--local 256] [--prec f32] [--set key=val ...]
"""
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
    p.add_argument("--prec", default="f32")
    p.add_argument("--reps", type=int, default=20)
    p.add_argument("--set", nargs="*", default=[])
    a = p.parse_args()
    import torch
    from paper_2507_11512_b200 import _lib
    from paper_2507_11512_b200.bench import BenchConfig, _build_state
    from paper_2507_11512_b200.krylov import GmresWorkspace, spmv
    from paper_2507_11512_b200.multigrid import fused_residual_restrict, prolong_add
    from paper_2507_11512_b200.smoother import forward_gs_sweep
    cfg = BenchConfig(local_nx=a.local, local_ny=a.local, local_nz=a.local, time_seconds=0)
    hier, lv0, b = _build_state(cfg, 1, None, 0)
    ctx = hier.ctx
    for kv in a.set:
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    lo = a.prec == "f32"
    dt = torch.float32 if lo else torch.float64
    st = ctx.stream

    def timeit(fn, reps=a.reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return round(e0.elapsed_time(e1) / reps * 1e3, 1)

    out = {"local": a.local, "prec": a.prec, "set": a.set}
    total = 0.0
    for l, lv in enumerate(hier.levels):
        A = lv.A_lo if lo else lv.A_hi
        n, ne = A.n_rows, A.n_cols_extended
        r = torch.randn(n, device="cuda", dtype=dt)
        z = torch.zeros(ne, device="cuda", dtype=dt)
        t0 = timeit(lambda: forward_gs_sweep(A, r, z, z_is_zero=True))
        t1 = timeit(lambda: forward_gs_sweep(A, r, z))
        out[f"L{l}_zero_sweep"] = t0
        out[f"L{l}_sweep"] = t1
        last = l == len(hier.levels) - 1
        total += t0 if last else t0 + t1
        if not last:
            nxt = hier.levels[l + 1]
            rc = torch.empty(nxt.A_hi.n_rows, device="cuda", dtype=dt)
            zc = torch.randn(nxt.A_hi.n_rows, device="cuda", dtype=dt)
            out[f"L{l}_restrict"] = timeit(lambda: fused_residual_restrict(A, r, z, nxt.f2c, out=rc))
            out[f"L{l}_prolong"] = timeit(lambda: prolong_add(z, zc, nxt.f2c))
            total += out[f"L{l}_restrict"] + out[f"L{l}_prolong"]
    out["sum_of_parts"] = round(total, 1)
    r0 = torch.randn(lv0.A_hi.n_rows, device="cuda", dtype=dt)
    out["vcycle"] = timeit(lambda: hier.apply(r0))
    A = lv0.A_lo if lo else lv0.A_hi
    x = torch.randn(A.n_cols_extended, device="cuda", dtype=dt)
    y = torch.empty(A.n_rows, device="cuda", dtype=dt)
    out["spmv"] = timeit(lambda: spmv(A, x, out=y))
    n = A.n_rows
    ws = GmresWorkspace.allocate(n, 30, np.float32 if lo else np.float64, device="cuda")
    ws.Q.normal_()
    w = torch.randn(-(-n // 32) * 32, device="cuda", dtype=dt)[:n]
    res = np.zeros(64)
    prec = _lib.F32 if lo else _lib.F64
    for k in (0, 14, 29):
        out[f"cgs2_kb{k + 1}"] = timeit(lambda: ctx.call("hpg_cgs2", prec, _lib.ptr(ws.Q), ws.Q.stride(0), k,
                                                          _lib.ptr(w), _lib.ptr(ws.Q[k + 1]),
                                                          res.ctypes.data_as(C.POINTER(C.c_double))), reps=5)
    hier.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
