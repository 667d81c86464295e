"""Reduction-order envelope of the mixed-precision iteration counts.

The reference's fp32 dot products and GEMVs go through OpenBLAS, whose
summation order is one of many legitimate fp32 orders; the inner iteration
count of the later GMRES-IR restart cycles moves by +-2 between such orders
(SURVEY.md 0.8).  This script runs the ORACLE (oracle/hpgmxp_oracle.py, pinned
bitwise to the reference by tests/test_oracle.py; its numpy GEMV path is the
reference's) with the CGS2 / norm reductions re-expressed in several fp32
orders and one fp64-accumulated order, and records the per-cycle counts:

  blas_gemv  the reference's own expressions (Q @ w, Q.T @ h: OpenBLAS sgemv)
  blas_dot   one OpenBLAS sdot per basis row
  pairwise   numpy pairwise fp32 summation
  lanes1/4/8 1, 4, 8 sequential fp32 accumulators (a naive loop, SIMD-like lanes)
  f64        fp64 accumulation, rounded to fp32 once (what libhpgmxp does)

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_envelope.py   (minutes)

writes tests/golden/reduction_envelope.json.  Test infrastructure only.
"""

import inspect
import json
import os
import sys
import textwrap
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))

CASES = {  # name: (local L, ranks, process grid, levels, m)
    "l16": (16, 1, None, 4, 30), "l32": (32, 1, None, 4, 30), "l4m5": (4, 1, None, 3, 5),
    "r2l16": (16, 2, None, 4, 30), "r8l8": (8, 8, None, 4, 30),
    "x211l16": (16, 2, (2, 1, 1), 4, 30), "x221l8": (8, 4, (2, 2, 1), 4, 30), "x212l8": (8, 4, (2, 1, 2), 4, 30),
}
VARIANTS = ("blas_gemv", "blas_dot", "pairwise", "lanes1", "lanes4", "lanes8", "f64")
F32 = np.float32


def _solve(variant, case):
    import hpgmxp_oracle as O
    L, R, dims, levels, m = CASES[case]

    def local_dot(a, b):
        if a.dtype != F32 or variant == "blas_dot":
            return a @ b
        if variant == "f64":
            return np.dot(a.astype(np.float64), b.astype(np.float64))
        if variant == "pairwise":
            return np.sum(a * b, dtype=F32)
        lanes = int(variant[5:])
        p = (a * b).astype(F32)
        p = np.concatenate([p, np.zeros((-len(p)) % lanes, F32)]).reshape(-1, lanes)
        acc = np.zeros(lanes, F32)
        for row in p:
            acc = acc + row
        out = F32(0)
        for v in acc:
            out = F32(out + v)
        return out

    def dots(Q, w, kb, Rk):
        parts = [np.array([local_dot(Q[q][j], w[q]) for j in range(kb)]) for q in range(Rk)]
        acc = parts[0].copy()
        for p in parts[1:]:
            acc = acc + p
        return acc.astype(F32) if Q[0].dtype == F32 else acc

    def norm2(w):
        acc = local_dot(w[0], w[0])
        for x in w[1:]:
            acc = acc + local_dot(x, x)
        return F32(acc) if w[0].dtype == F32 else acc

    src = inspect.getsource(O.Solver.gmres)
    if variant != "blas_gemv":
        src = src.replace("self.world.allreduce([Q[q][:kb] @ w[q] for q in range(R)])", "DOTS(Q, w, kb, R)")
        src = src.replace("np.sqrt(self.world.allreduce([ww @ ww for ww in w]))", "np.sqrt(NORM2(w))")
    ns = dict(O.__dict__)
    ns.update(DOTS=dots, NORM2=norm2)
    exec(textwrap.dedent(src), ns)
    s = O.Solver(L, L, L, R, levels, dims=dims)
    res, _ = ns["gmres"](s, s.rhs(), "mixed", 1e-9, 300, m)
    return variant, case, res["cycle_iters"]


def main():
    jobs = [(v, c) for c in CASES for v in VARIANTS]
    out = {c: {} for c in CASES}
    with ProcessPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
        for v, c, cyc in ex.map(_solve, *zip(*jobs)):
            out[c][v] = cyc
            print(c, v, cyc, flush=True)
    with open(os.path.join(HERE, "reduction_envelope.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
