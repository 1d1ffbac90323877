"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys


def rows(path):
    out, hdr = [], None
    for r in csv.reader(open(path)):
        if 'Kernel Name' in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get('Metric Name') == 'gpu__time_duration.sum':
                v = float(d['Metric Value'].replace(',', ''))
                unit = d['Metric Unit']
                us = v / 1000 if unit == 'ns' else v * 1000 if unit == 'ms' else v
                out.append((int(d['ID']), d['Kernel Name'], us))
    return out


if __name__ == "__main__":
    for path in sys.argv[1:]:
        print(path)
        for i, name, us in rows(path):
            print(f"  {i:3d} {us:10.1f} us  {name[:110]}")
