"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`): per-kernel count,
total and mean time, and share of the captured region."""
import collections
import csv
import sys


def summarise(path, top=40):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(',', ''))
        except ValueError:
            continue
        scale = {'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'nsecond': 1e-3}.get(r[ui], 1e-3)
        n = r[ki].split('(')[0].replace('void ', '').replace('pdipc::', '')
        agg[n][0] += 1
        agg[n][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    out = [f"{'kernel':44s} {'launches':>8s} {'total_us':>10s} {'us/launch':>10s} {'share':>6s}"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{n[:44]:44s} {c:8d} {t:10.1f} {t / c:10.2f} {100 * t / tot:5.1f}%")
    out.append(f"total {sum(v[0] for v in agg.values())} launches, {tot:.1f} us (serialised, cold)")
    return "\n".join(out)


if __name__ == '__main__':
    print(summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40))
