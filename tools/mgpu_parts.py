"""Per-motif seconds of one 30-iteration mixed restart cycle at L^3 per rank under
torchrun (library CUDA events), rank 0 prints.  Tuning aid, not a bench number."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    import torch
    from paper_2507_11512_b200.bench import BenchConfig, _build_state, _solve
    from paper_2507_11512_b200.comm import World
    from paper_2507_11512_b200.metrics import Tally
    world = World()
    R = world.nranks
    cfg = BenchConfig(local_nx=L, local_ny=L, local_nz=L, ranks=R, time_seconds=0)
    hier, lv, b = _build_state(cfg, R, world if R > 1 else None, world.rank)
    w = world if R > 1 else None
    _solve(cfg, hier, lv, b, w, world.rank, "mixed", 1e-9, 30)
    torch.cuda.synchronize()
    world.barrier()
    tal = Tally()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(hier.ctx.stream)
    _solve(cfg, hier, lv, b, w, world.rank, "mixed", 1e-9, 30, tal)
    e1.record(hier.ctx.stream)
    torch.cuda.synchronize()
    out = {"rank": world.rank, "ranks": R, "ms": e0.elapsed_time(e1),
           "motif_ms": {k: round(v * 1e3, 2) for k, v in tal.seconds.items()}}
    allo = world.gather(world.rank, out)
    if world.rank == 0:
        for o in allo:
            print(json.dumps(o))
    hier.close()


if __name__ == "__main__":
    main()
