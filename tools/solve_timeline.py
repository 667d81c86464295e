"""Kernel timeline of one warm mixed solve at L^3 (torch.profiler / CUPTI
activity records): busy time per kernel, device idle gaps and what precedes
them.  Tells whether the solve is kernel-bound or waits on the host.

    python tools/solve_timeline.py [--local 256] [--out gpurun_out/timeline.json]
    torchrun --nproc-per-node N tools/solve_timeline.py   (one file per rank)
"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--local", type=int, default=256)
    p.add_argument("--mode", default="mixed")
    p.add_argument("--out", default="gpurun_out/timeline.json")
    a = p.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_2507_11512_b200.bench import BenchConfig, _build_state, _solve
    from paper_2507_11512_b200.comm import World
    L = a.local
    nr = int(os.environ.get("WORLD_SIZE", "1"))
    world = World() if nr > 1 else None
    rank = world.rank if world else 0
    cfg = BenchConfig(local_nx=L, local_ny=L, local_nz=L, ranks=nr, time_seconds=0)
    hier, lv, b = _build_state(cfg, nr, world, rank)
    for _ in range(2):
        _solve(cfg, hier, lv, b, world, rank, a.mode, cfg.tol, cfg.max_iters)
    torch.cuda.synchronize()
    if world:
        world.barrier()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        res = _solve(cfg, hier, lv, b, world, rank, a.mode, cfg.tol, cfg.max_iters)
        torch.cuda.synchronize()
    if nr > 1:
        a.out = a.out.replace(".json", f"_rank{rank}.json")
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in ev), key=lambda x: x[0])
    busy = collections.defaultdict(float)
    count = collections.Counter()
    for s, e, n in ks:
        short = n.split("(")[0][:80]
        busy[short] += e - s
        count[short] += 1
    span = ks[-1][1] - ks[0][0]
    gaps = []
    end = ks[0][1]
    for i in range(1, len(ks)):
        s, e, n = ks[i]
        if s > end:
            gaps.append((s - end, ks[i - 1][2].split("(")[0][:60], n.split("(")[0][:60]))
        end = max(end, e)
    gap_total = sum(g[0] for g in gaps)
    by_pair = collections.defaultdict(lambda: [0.0, 0])
    for g, a1, b1 in gaps:
        by_pair[(a1, b1)][0] += g
        by_pair[(a1, b1)][1] += 1
    out = {
        "iterations": res.iterations,
        "span_us": round(span, 1),
        "kernels": len(ks),
        "busy_us": round(sum(busy.values()), 1),
        "idle_us": round(gap_total, 1),
        "per_kernel": sorted(([k, count[k], round(v, 1)] for k, v in busy.items()), key=lambda x: -x[2]),
        "gaps_by_pair": sorted(([a1, b1, round(v[0], 1), v[1]] for (a1, b1), v in by_pair.items()),
                               key=lambda x: -x[2])[:25],
    }
    # note: a PDL kernel's duration starts at its early launch (it waits on the device
    # for its predecessor), so per-kernel sums over-count; span and idle are exact
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("iterations", "span_us", "kernels", "busy_us", "idle_us")}))
    for row in out["per_kernel"][:20]:
        print(row)
    for row in out["gaps_by_pair"][:15]:
        print("gap", row)
    hier.close()


if __name__ == "__main__":
    main()
