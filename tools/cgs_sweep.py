"""Time the fused CGS2 step for every (WR, RPW, U) configuration at several basis
sizes kb (fp32 256^3 vectors, CUDA events).  Tuning aid for cgs_config's table."""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODES = [int(c) for c in os.environ["CGS_CODES"].split(",")] if os.environ.get("CGS_CODES") else [118, 218, 418, 818, 424, 824, 422, 432, 832, 442, 842, 441, 242, 281, 461, 861, 481, 881,
         3441, 3841, 3831, 3422, 3822]  # 3xxx: built for 3 CTAs per SM


def main():
    import torch
    from paper_2507_11512_b200 import _lib
    from paper_2507_11512_b200.geometry import GlobalProblem
    from paper_2507_11512_b200.krylov import GmresWorkspace
    from paper_2507_11512_b200.multigrid import build_hierarchy
    prec = sys.argv[1] if len(sys.argv) > 1 else "f32"
    hier = build_hierarchy(GlobalProblem.from_local(256, 256, 256, 1).domain(0), 1)
    ctx = hier.ctx
    n = hier.levels[0].A_hi.n_rows
    dt = np.float32 if prec == "f32" else np.float64
    tdt = torch.float32 if prec == "f32" else torch.float64
    P = _lib.F32 if prec == "f32" else _lib.F64
    ws = GmresWorkspace.allocate(n, 30, dt, device="cuda")
    ws.Q.normal_()
    w = torch.randn(-(-n // 32) * 32, device="cuda", dtype=tdt)[:n]
    res = np.zeros(64)
    st = ctx.stream
    out = {}
    kbs = [int(x) for x in os.environ.get("CGS_KBS", "1,2,4,6,8,12,16,20,24,28,30").split(",")]
    for kb in kbs:
        row = {}
        for code in [0] + CODES:
            wr, rpw = (code % 1000) // 100, (code // 10) % 10
            if code and wr * rpw < kb:
                continue
            ctx.set_option("cgs_cfg", code)
            k = kb - 1
            f = lambda: ctx.call("hpg_cgs2", P, _lib.ptr(ws.Q), ws.Q.stride(0), k, _lib.ptr(w), _lib.ptr(ws.Q[kb]),
                                 res.ctypes.data_as(C.POINTER(C.c_double)))
            f()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(5):
                f()
            e1.record(st)
            torch.cuda.synchronize()
            row[code] = round(e0.elapsed_time(e1) / 5 * 1e3, 1)
        best = min((v, c) for c, v in row.items() if c)
        out[kb] = {"table": row[0], "best": best[1], "best_us": best[0]}
        if os.environ.get("CGS_ROWS"):
            out[kb]["all"] = row
        print(kb, out[kb], flush=True)
    print(json.dumps(out))
    hier.close()


if __name__ == "__main__":
    main()
