"""A few level-0 fp32 (or fp64) forward sweeps at L^3 -- the target of an ncu capture.

    python tools/one_sweep.py [--local 256] [--prec f32] [--zero] [--reps 3] [--set key=val ...]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--local", type=int, default=256)
    p.add_argument("--prec", default="f32")
    p.add_argument("--zero", action="store_true")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--what", default="sweep", choices=("sweep", "spmv", "vcycle"))
    p.add_argument("--set", nargs="*", default=[])
    a = p.parse_args()
    import torch
    from paper_2507_11512_b200.bench import BenchConfig, _build_state
    from paper_2507_11512_b200.krylov import spmv
    from paper_2507_11512_b200.smoother import forward_gs_sweep
    cfg = BenchConfig(local_nx=a.local, local_ny=a.local, local_nz=a.local, time_seconds=0)
    hier, lv, b = _build_state(cfg, 1, None, 0)
    for kv in a.set:
        k, v = kv.split("=")
        hier.ctx.set_option(k, int(v))
    A = lv.A_lo if a.prec == "f32" else lv.A_hi
    dt = torch.float32 if a.prec == "f32" else torch.float64
    r = torch.randn(A.n_rows, device="cuda", dtype=dt)
    z = torch.zeros(A.n_cols_extended, device="cuda", dtype=dt)
    y = torch.empty(A.n_rows, device="cuda", dtype=dt)
    for _ in range(a.reps):
        if a.what == "sweep":
            forward_gs_sweep(A, r, z, z_is_zero=a.zero)
        elif a.what == "spmv":
            spmv(A, z, out=y)
        else:
            hier.apply(r)
    torch.cuda.synchronize()
    hier.close()
    print("ok")


if __name__ == "__main__":
    main()
