"""Same-box A/B of whole mixed solves at L^3 under option settings, interleaved
(A B A B ...), CUDA events on the solve stream.  Each setting must take the same
iteration count.  Not a bench number.

    python tools/solve_ab.py [--local 256] [--rounds 3] --opt cgs_hint:0,1,2,3
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--local", type=int, default=256)
    p.add_argument("--rounds", type=int, default=3)
    p.add_argument("--opt", required=True, help="option:v0,v1,...")
    p.add_argument("--mode", default="mixed")
    a = p.parse_args()
    import torch
    from paper_2507_11512_b200.bench import BenchConfig, _build_state, _solve
    from paper_2507_11512_b200.comm import runtime
    L = a.local
    cfg = BenchConfig(local_nx=L, local_ny=L, local_nz=L, time_seconds=0)
    hier, lv, b = _build_state(cfg, 1, None, 0)
    ctx = hier.ctx
    stream = runtime().stream
    key, vals = a.opt.split(":")
    vals = [int(v) for v in vals.split(",")]
    times = {v: [] for v in vals}
    iters = {}
    for v in vals:  # warm every setting (graph capture)
        ctx.set_option(key, v)
        _solve(cfg, hier, lv, b, None, 0, a.mode, cfg.tol, cfg.max_iters)
    for _ in range(a.rounds):
        for v in vals:
            ctx.set_option(key, v)
            _solve(cfg, hier, lv, b, None, 0, a.mode, cfg.tol, cfg.max_iters)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = _solve(cfg, hier, lv, b, None, 0, a.mode, cfg.tol, cfg.max_iters)
            e1.record(stream)
            torch.cuda.synchronize()
            times[v].append(round(e0.elapsed_time(e1), 2))
            iters.setdefault(v, res.iterations)
            if res.iterations != iters[v]:
                raise RuntimeError(f"{key}={v}: iterations changed {iters[v]} -> {res.iterations}")
    out = {"local": L, "opt": key, "mode": a.mode, "iters": iters, "ms": times,
           "best_ms": {v: min(t) for v, t in times.items()}}
    print(json.dumps(out))
    hier.close()


if __name__ == "__main__":
    main()
