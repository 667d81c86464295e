"""Print per-restart-cycle GMRES iteration counts of the device solver next to
the reference envelope (tests/golden/solves.json) for the single-rank cases.

    python tools/cycle_counts.py            (on a GPU box)
"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = {"l16": (16, 4, 30), "l32": (32, 4, 30), "l4m5": (4, 3, 5)}


def main():
    from paper_2507_11512_b200.geometry import GlobalProblem
    from paper_2507_11512_b200.krylov import gmres_solve
    from paper_2507_11512_b200.multigrid import build_hierarchy
    from paper_2507_11512_b200.problem import generate_rhs
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "solves.json")))
    for case, (l, levels, m) in CASES.items():
        h = build_hierarchy(GlobalProblem.from_local(l, l, l, 1).domain(0), levels)
        lv = h.levels[0]
        b = generate_rhs(lv.A_hi).b
        for mode in ("double", "mixed"):
            x = np.zeros(lv.A_hi.n_rows)
            res = gmres_solve(lv.A_hi, lv.A_lo, h.preconditioner(), b, x0=x, mode=mode, m=m)
            env = {th: gold[case][th][mode]["cycle_iters"] for th in ("1", "default")}
            print(f"{case} {mode}: gpu {res.cycle_iterations} (total {res.iterations}, relres "
                  f"{res.relres:.3e})  reference {env}", flush=True)
        h.close()


if __name__ == "__main__":
    main()
