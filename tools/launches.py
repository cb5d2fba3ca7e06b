"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import csv
import sys


def main(path, top=14):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if 'Kernel Name' in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get('Metric Name') == 'gpu__time_duration.sum':
                out.append((d['Kernel Name'].split('(')[0][:60], float(d['Metric Value'])))
    tot = sum(v for _, v in out)
    agg, cnt = {}, {}
    for k, v in out:
        agg[k] = agg.get(k, 0) + v
        cnt[k] = cnt.get(k, 0) + 1
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"{v / 1e6:9.3f} ms {100 * v / tot:6.2f}% n={cnt[k]:4d} {k}")
    print(f"{len(out)} launches, total {tot / 1e6:.3f} ms (serialised, cold-cache)")


if __name__ == "__main__":
    main(sys.argv[1])
