"""ncu target: one V-cycle (f32), one CGS2 at k=29 (f32), one SpMV (f32), one fp64
residual, between cudaProfilerStart/Stop, after a warm-up of each."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    import torch
    from paper_2507_11512_b200 import _lib
    from paper_2507_11512_b200.bench import BenchConfig, _build_state
    from paper_2507_11512_b200.krylov import GmresWorkspace
    cfg = BenchConfig(local_nx=L, local_ny=L, local_nz=L, time_seconds=0)
    hier, lv, b = _build_state(cfg, 1, None, 0)
    ctx = hier.ctx
    n, ne = lv.A_hi.n_rows, lv.A_hi.n_cols_extended
    ws = GmresWorkspace.allocate(n, 30, np.float32, device="cuda")
    ws.Q.normal_()
    w = torch.randn(n, device="cuda")
    z = torch.zeros(ne, device="cuda")
    y = torch.empty(n, device="cuda")
    x64 = torch.randn(ne, device="cuda", dtype=torch.float64)
    r64 = torch.empty(n, device="cuda", dtype=torch.float64)
    res = np.zeros(64)
    rho = C.c_double()

    def once():
        hier.apply(ws.Q[3], out=z)
        ctx.call("hpg_cgs2", _lib.F32, _lib.ptr(ws.Q), ws.Q.stride(0), 29, _lib.ptr(w),
                 _lib.ptr(ws.Q[30]), res.ctypes.data_as(C.POINTER(C.c_double)))
        ctx.call("hpg_spmv", 0, _lib.F32, _lib.ptr(z), _lib.ptr(y))
        ctx.call("hpg_residual", _lib.ptr(b), _lib.ptr(x64), _lib.ptr(r64), C.byref(rho))

    once()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    once()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("ok")
    hier.close()


if __name__ == "__main__":
    main()
