"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if 'Kernel Name' in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d['Metric Name'] != 'gpu__time_duration.sum':
            continue
        v = float(d['Metric Value'].replace(',', ''))
        unit = d['Metric Unit']
        v = v / 1000.0 if unit in ('nsecond', 'ns') else v * 1000.0 if unit in ('msecond', 'ms') else v
        name = d['Kernel Name'].split('(')[0][-70:]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'total us':>10} {'share':>6} {'launches':>8} {'avg us':>9}  kernel")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f'{t:10.1f} {100 * t / tot:5.1f}% {c:8d} {t / c:9.2f}  {k}')
    print(f'{tot:10.1f} total (us, serialised cold-cache ncu times)')


if __name__ == '__main__':
    main(sys.argv[1])
