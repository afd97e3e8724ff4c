"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel name."""
import collections
import csv
import sys


def summarize(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hi]
    ki, mi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        name = r[ki].split('(')[0][:70]
        v = float(r[mi].replace(',', ''))
        v *= {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"{'kernel':70s} {'launches':>8s} {'total_us':>11s} {'avg_us':>9s} {'share':>6s}"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{n:70s} {c:8d} {t:11.1f} {t / c:9.2f} {100 * t / tot:5.1f}%")
    out.append(f"total {tot / 1e3:.2f} ms over {sum(v[0] for v in agg.values())} launches")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
