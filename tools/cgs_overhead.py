"""Fixed cost of one fused CGS2 call (grid barriers, folds, launch): time it on a
tiny vector (L^3 rows, default 16^3) where streaming is negligible.  Not a bench number.

    python tools/cgs_overhead.py [L] [--set key=val ...]
"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    args = [a for a in sys.argv[1:] if "=" not in a]
    sets = [a for a in sys.argv[1:] if "=" in a]
    L = int(args[0]) if args else 16
    import torch
    from paper_2507_11512_b200 import _lib
    from paper_2507_11512_b200.geometry import GlobalProblem
    from paper_2507_11512_b200.krylov import GmresWorkspace
    from paper_2507_11512_b200.multigrid import build_hierarchy
    hier = build_hierarchy(GlobalProblem.from_local(L, L, L, 1).domain(0), 2)
    ctx = hier.ctx
    for kv in sets:
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    n = hier.levels[0].A_hi.n_rows
    ws = GmresWorkspace.allocate(n, 30, np.float32, device="cuda")
    ws.Q.normal_()
    w = torch.randn(-(-n // 32) * 32, device="cuda")[:n]
    res = np.zeros(64)
    st = ctx.stream
    out = {"n": n, "set": sets}
    for kb in (1, 8, 16, 30):
        f = lambda: ctx.call("hpg_cgs2", _lib.F32, _lib.ptr(ws.Q), ws.Q.stride(0), kb - 1, _lib.ptr(w),
                             _lib.ptr(ws.Q[kb]), res.ctypes.data_as(C.POINTER(C.c_double)))
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(50):
            ctx.call("hpg_cgs2_begin", _lib.F32, _lib.ptr(ws.Q), ws.Q.stride(0), kb - 1, _lib.ptr(w),
                     _lib.ptr(ws.Q[kb]))
        e1.record(st)
        torch.cuda.synchronize()
        out[f"kb{kb}_us"] = round(e0.elapsed_time(e1) / 50 * 1e3, 1)
    print(json.dumps(out))
    hier.close()


if __name__ == "__main__":
    main()
