"""Latency of one halo exchange (each level, fp32) and one rank-ordered all-reduce
under torchrun, back-to-back calls timed with CUDA events.  Tuning aid."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    import torch
    from paper_2507_11512_b200 import _lib
    from paper_2507_11512_b200.comm import World
    from paper_2507_11512_b200.geometry import GlobalProblem
    from paper_2507_11512_b200.multigrid import build_hierarchy
    world = World()
    R = world.nranks
    h = build_hierarchy(GlobalProblem.from_local(L, L, L, R).domain(world.rank), 4, world, world.rank)
    ctx = h.ctx
    out = {"rank": world.rank, "p2p": ctx.p2p}
    for li, lv in enumerate(h.levels):
        v = torch.zeros(lv.A_hi.n_cols_extended, device="cuda")
        for _ in range(3):
            ctx.call("hpg_exchange", li, _lib.F32, _lib.ptr(v))
        torch.cuda.synchronize()
        world.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        for _ in range(50):
            ctx.call("hpg_exchange", li, _lib.F32, _lib.ptr(v))
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        out[f"exchange_L{li}_us"] = round(e0.elapsed_time(e1) / 50 * 1e3, 2)
    # level-0 kernels that carry a collective: CGS2 (3 all-reduces), SpMV and a
    # GS sweep (one exchange each), back to back
    import numpy as np
    from paper_2507_11512_b200.krylov import GmresWorkspace
    lv = h.levels[0]
    n, ne = lv.A_hi.n_rows, lv.A_hi.n_cols_extended
    ws = GmresWorkspace.allocate(n, 30, np.float32, device="cuda")
    ws.Q.normal_()
    w = torch.randn(-(-n // 32) * 32, device="cuda")[:n]
    res = np.zeros(64)
    x = torch.randn(ne, device="cuda")
    y = torch.empty(n, device="cuda")

    def timeit(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        world.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        for _ in range(reps):
            fn()
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        return round(e0.elapsed_time(e1) / reps * 1e3, 1)
    for k in (0, 15, 29):
        out[f"cgs2_kb{k + 1}_us"] = timeit(lambda: ctx.call(
            "hpg_cgs2", _lib.F32, _lib.ptr(ws.Q), ws.Q.stride(0), k, _lib.ptr(w), _lib.ptr(ws.Q[k + 1]),
            res.ctypes.data_as(C.POINTER(C.c_double))))
    out["spmv_L0_us"] = timeit(lambda: ctx.call("hpg_spmv", 0, _lib.F32, _lib.ptr(x), _lib.ptr(y)))
    out["gs_sweep_L0_us"] = timeit(lambda: ctx.call("hpg_gs_sweep", 0, _lib.F32, _lib.ptr(y), _lib.ptr(x), 0))
    vals = (C.c_double * 4)(1, 2, 3, 4)
    world.barrier()
    import time
    t0 = time.perf_counter()
    for _ in range(50):
        ctx.call("hpg_allreduce_host", vals, 4)
    out["allreduce_host_roundtrip_us"] = round((time.perf_counter() - t0) / 50 * 1e6, 2)
    allo = world.gather(world.rank, out)
    if world.rank == 0:
        for o in allo:
            print(json.dumps(o))
    h.close()


if __name__ == "__main__":
    main()
