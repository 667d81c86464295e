"""Small driver for ncu: one warm-up and one timed mixed (or double) GMRES-IR
solve at L^3, capped at --iters inner iterations.  Not a bench number."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--local", type=int, default=256)
    p.add_argument("--iters", type=int, default=30)
    p.add_argument("--mode", default="mixed")
    p.add_argument("--warm", type=int, default=1)
    a = p.parse_args()
    import torch
    from paper_2507_11512_b200.bench import BenchConfig, _build_state, _solve
    cfg = BenchConfig(local_nx=a.local, local_ny=a.local, local_nz=a.local, time_seconds=0)
    hier, lv, b = _build_state(cfg, 1, None, 0)
    for _ in range(a.warm):
        _solve(cfg, hier, lv, b, None, 0, a.mode, 1e-9, a.iters)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    res = _solve(cfg, hier, lv, b, None, 0, a.mode, 1e-9, a.iters)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("iterations", res.iterations, "relres", res.relres, "launches", hier.ctx.launches())
    hier.close()


if __name__ == "__main__":
    main()
