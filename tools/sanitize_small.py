"""Small end-to-end run for compute-sanitizer (one tool per call): 16^3 hierarchy,
V-cycles in both precisions, fused CGS2 at several k, a mixed and a double solve."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2507_11512_b200 import _lib
    from paper_2507_11512_b200.bench import BenchConfig, _build_state, _solve
    from paper_2507_11512_b200.krylov import GmresWorkspace
    cfg = BenchConfig(local_nx=16, local_ny=16, local_nz=16, time_seconds=0)
    hier, lv, b = _build_state(cfg, 1, None, 0)
    n = lv.A_hi.n_rows
    for mode in ("mixed", "double"):
        r = _solve(cfg, hier, lv, b, None, 0, mode, 1e-9, 300)
        print(mode, r.iterations, r.relres)
    ws = GmresWorkspace.allocate(n, 30, np.float32, device="cuda")
    ws.Q.normal_()
    w = torch.randn(-(-n // 32) * 32, device="cuda")[:n]
    out = np.zeros(64)
    for k in (0, 3, 9, 20, 29):
        hier.ctx.call("hpg_cgs2", _lib.F32, _lib.ptr(ws.Q), ws.Q.stride(0), k, _lib.ptr(w),
                      _lib.ptr(ws.Q[k + 1]), out.ctypes.data_as(C.POINTER(C.c_double)))
    hier.ctx.set_option("tail_rows", 1 << 30)
    hier.apply(torch.randn(n, device="cuda"))
    torch.cuda.synchronize()
    hier.close()
    # the tensor-copy staged kernels (colour passes, brick passes, SpMV, residual)
    # on every level that admits them, at 32^3
    cfg = BenchConfig(local_nx=32, local_ny=32, local_nz=32, time_seconds=0)
    hier, lv, b = _build_state(cfg, 1, None, 0)
    for brick in (0, 3):
        hier.ctx.set_option("tma_min_rows", 0)
        hier.ctx.set_option("brick", brick)
        for mode in ("mixed", "double"):
            r = _solve(cfg, hier, lv, b, None, 0, mode, 1e-9, 40)
            print("tma", brick, mode, r.iterations, r.relres)
    torch.cuda.synchronize()
    hier.close()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
