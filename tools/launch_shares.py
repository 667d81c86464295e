"""Per-kernel shares of an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv): launches, summed and average
time, share, DRAM bytes per launch -- as a markdown table.

    python tools/launch_shares.py gpurun_out/r02l_launches.csv
"""
import collections
import csv
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "").replace("hpg::", "")
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0) / 1e3  # ns -> us
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    total = sum(a[1] for a in agg.values())
    print(f"{len(per)} launches, {total:.1f} us summed.\n")
    print("| kernel | launches | sum us | share | avg us | DRAM MB / launch |")
    print("|---|---|---|---|---|---|")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {t:.1f} | {100 * t / total:.1f}% | {t / n:.1f} | {b / n / 1e6:.1f} |")


if __name__ == "__main__":
    main()
