"""Same-box A/B of the level-0 sweep and V-cycle kernels at L^3 (CUDA events,
warm, repeated), option pairs interleaved; also checks that each variant
produces the same bits.  Not a bench number.

    python tools/sweep_ab.py [--local 256] [--reps 20] [--opt tma:0,3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--local", type=int, default=256)
    p.add_argument("--reps", type=int, default=20)
    p.add_argument("--opt", default="tma:0,3", help="option:valueA,valueB")
    p.add_argument("--set", nargs="*", default=[], help="key=value options applied first")
    a = p.parse_args()
    import torch
    from paper_2507_11512_b200.bench import BenchConfig, _build_state
    from paper_2507_11512_b200.smoother import forward_gs_sweep
    cfg = BenchConfig(local_nx=a.local, local_ny=a.local, local_nz=a.local, time_seconds=0)
    hier, lv, b = _build_state(cfg, 1, None, 0)
    ctx = hier.ctx
    st = ctx.stream
    for kv in a.set:
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    n, ne = lv.A_hi.n_rows, lv.A_hi.n_cols_extended
    key, vals = a.opt.split(":")
    vals = [int(v) for v in vals.split(",")]
    gen = torch.Generator("cuda").manual_seed(1)
    r32 = torch.randn(n, device="cuda", generator=gen)
    r64 = r32.double()
    z32 = torch.zeros(ne, device="cuda")
    z64 = torch.zeros(ne, device="cuda", dtype=torch.float64)

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

    import ctypes as C
    from paper_2507_11512_b200 import _lib
    from paper_2507_11512_b200.krylov import spmv
    x32 = torch.randn(ne, device="cuda", generator=gen)
    x64 = x32.double()
    y32 = torch.empty(n, device="cuda")
    y64 = torch.empty(n, device="cuda", dtype=torch.float64)
    rho2 = C.c_double()
    cases = {
        "spmv_f32": lambda: spmv(lv.A_lo, x32, out=y32),
        "spmv_f64": lambda: spmv(lv.A_hi, x64, out=y64),
        "resid_f64": lambda: ctx.call("hpg_residual", _lib.ptr(b), _lib.ptr(x64), _lib.ptr(y64), C.byref(rho2)),
        "sweep_f32": lambda: forward_gs_sweep(lv.A_lo, r32, z32),
        "zero_sweep_f32": lambda: forward_gs_sweep(lv.A_lo, r32, z32, z_is_zero=True),
        "sweep_f64": lambda: forward_gs_sweep(lv.A_hi, r64, z64),
        "zero_sweep_f64": lambda: forward_gs_sweep(lv.A_hi, r64, z64, z_is_zero=True),
        "vcycle_f32": lambda: hier.apply(r32),
        "vcycle_f64": lambda: hier.apply(r64),
    }
    out = {"local": a.local, "option": key}
    bits = {}
    for rnd in range(2):
        for v in vals:
            ctx.set_option(key, v)
            for name, fn in cases.items():
                t = timeit(fn)
                out.setdefault(f"{name}_{key}{v}", []).append(round(t, 1))
    for v in vals:  # bitwise: two sweeps from zero + one V-cycle, each precision
        ctx.set_option(key, v)
        z32.zero_()
        z64.zero_()
        forward_gs_sweep(lv.A_lo, r32, z32, z_is_zero=True)
        forward_gs_sweep(lv.A_lo, r32, z32)
        forward_gs_sweep(lv.A_hi, r64, z64, z_is_zero=True)
        forward_gs_sweep(lv.A_hi, r64, z64)
        sp = (spmv(lv.A_lo, x32, out=y32).clone(), spmv(lv.A_hi, x64, out=y64).clone())
        ctx.call("hpg_residual", _lib.ptr(b), _lib.ptr(x64), _lib.ptr(y64), C.byref(rho2))
        bits[v] = (z32.clone(), z64.clone(), hier.apply(r32).clone(), hier.apply(r64).clone()) + sp + (y64.clone(),)
        out.setdefault("rho2", []).append(rho2.value)
    ref = bits[vals[0]]
    out["bitwise_equal"] = all(all(torch.equal(x, y) for x, y in zip(ref, bits[v])) for v in vals[1:])
    hier.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
