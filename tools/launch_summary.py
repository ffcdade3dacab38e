# SPDX-License-Identifier: Apache-2.0
"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv),
over the last `frac` of the launches (solve_timeline.py: the last of three solves).

    python tools/launch_summary.py LIST.csv [frac=0.3333]
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    frac = float(sys.argv[2]) if len(sys.argv) > 2 else 1 / 3
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h, data = rows[0], rows[1:]
    iN, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    last = data[int(len(data) * (1 - frac)):]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in last:
        v = float(r[iV].replace(",", "")) * {"usecond": 1e3, "msecond": 1e6}.get(r[iU], 1)
        nm = r[iN].split("(")[0][:70]
        agg[nm][0] += 1
        agg[nm][1] += v
    tot = sum(v for _, v in agg.values())
    print(f"{path}: {len(last)} launches, {tot / 1e6:.2f} ms")
    for nm, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {c:6d} {v / 1e6:9.2f} ms {100 * v / tot:5.1f}%  avg {v / c / 1e3:8.1f} us  {nm}")


if __name__ == "__main__":
    main()
