"""ncu target: fused and per-pass CGS2 at several kb (f32, 256^3-sized vectors)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    ks = [int(k) for k in sys.argv[2].split(",")] if len(sys.argv) > 2 else [29]
    import torch
    from paper_2507_11512_b200 import _lib
    from paper_2507_11512_b200.geometry import GlobalProblem
    from paper_2507_11512_b200.krylov import GmresWorkspace
    from paper_2507_11512_b200.multigrid import build_hierarchy
    hier = build_hierarchy(GlobalProblem.from_local(L, L, L, 1).domain(0), 1)
    ctx = hier.ctx
    n = hier.levels[0].A_hi.n_rows
    ws = GmresWorkspace.allocate(n, 30, np.float32, device="cuda")
    ws.Q.normal_()
    w = torch.randn(-(-n // 32) * 32, device="cuda")[:n]
    res = np.zeros(64)
    st = ctx.stream

    def run(k):
        ctx.call("hpg_cgs2", _lib.F32, _lib.ptr(ws.Q), ws.Q.stride(0), k, _lib.ptr(w),
                 _lib.ptr(ws.Q[k + 1]), res.ctypes.data_as(C.POINTER(C.c_double)))

    for fused in (1, 0):
        ctx.set_option("cgs_fused", fused)
        for k in ks:
            run(k)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(5):
                run(k)
            e1.record(st)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 5 * 1e3
            kb = k + 1
            print(f"fused={fused} kb={kb} {us:.1f} us  actual~{(3*kb*n*4 + 6*n*4)/us/1e3:.0f} GB/s"
                  f"  model {(4*n*kb*4 + 4*n*4 + 3*n*4)/us/1e3:.0f} GB/s")
    torch.cuda.cudart().cudaProfilerStart()
    ctx.set_option("cgs_fused", 1)
    run(ks[-1])
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    hier.close()


if __name__ == "__main__":
    main()
