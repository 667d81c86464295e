"""Summarise an ncu launch list (csv) and/or an ncu --set full report into markdown.

    python tools/summarize_ncu.py --launches L.csv [--report R.ncu-rep] > profiles/rNN_summary.md
"""
import argparse
import collections
import csv
import io
import subprocess


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, gi, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Grid Size", "Metric Name", "Metric Value", "ID"))
    per, names = collections.defaultdict(dict), {}
    for r in rows[1:]:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = (r[ki].split("(")[0].replace("void ", "").replace("hpg::", ""), r[gi])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for i, m in per.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a = agg[names[i]]
        a[0] += 1
        a[1] += t
        a[2] += b
        tot += t
    out = ["| kernel | grid | launches | total ms | share | avg us | DRAM GB/s (ncu, cold L2) |",
           "|---|---|---|---|---|---|---|"]
    for (k, g), (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {g} | {c} | {t/1e6:.2f} | {100*t/tot:.1f}% | {t/c/1e3:.1f} | {b/t if t else 0:.0f} |")
    out.append(f"\nTotal kernel time {tot/1e6:.2f} ms over {len(per)} launches.")
    return "\n".join(out)


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    want = [("gpu__time_duration.sum", "dur us"), ("dram__bytes_read.sum", "DRAM rd"),
            ("dram__bytes_write.sum", "DRAM wr"), ("launch__registers_per_thread", "regs"),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps act %"),
            ("launch__grid_size", "grid")]
    stalls = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled")]
    units = rows[1]
    out = ["| kernel | " + " | ".join(w[1] for w in want) + " | top stalls |",
           "|---|" + "---|" * (len(want) + 1)]
    for r in rows[2:]:
        vals = []
        for key, _ in want:
            if key in hdr:
                j = hdr.index(key)
                vals.append(f"{r[j]} {units[j]}".strip())
            else:
                vals.append("-")
        st = sorted(((float(r[i].replace(",", "")) if r[i] else 0.0,
                      hdr[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                     for i in stalls), reverse=True)[:3]
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("hpg::", "")
        out.append(f"| `{name[:48]}` | " + " | ".join(vals) + " | " +
                   ", ".join(f"{n} {v:.1f}" for v, n in st) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    a = ap.parse_args()
    if a.launches:
        print("### Launch list (ncu --metrics gpu__time_duration.sum,dram__bytes_*; serialised, cold cache)\n")
        print(launches(a.launches))
    if a.report:
        print("\n### ncu --set full, selected kernels\n")
        print(report(a.report))
