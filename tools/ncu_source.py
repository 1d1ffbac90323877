"""Per-opcode and per-instruction stall attribution from an ncu source page."""
import collections
import csv
import sys


def blocks(path):
    out, cur = [], None
    for l in open(path).read().splitlines():
        if l.startswith('"Kernel Name"'):
            cur = [l]
            out.append(cur)
        elif cur is not None:
            cur.append(l)
    return out


def main(path, k=0, top=25):
    b = blocks(path)[k]
    print(b[0][:150])
    rows = list(csv.reader(b[1:]))
    hdr = rows[0]
    reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
    si = hdr.index('Warp Stall Sampling (All Samples)')
    ie = hdr.index('Instructions Executed')
    agg = collections.defaultdict(collections.Counter)
    cnt = collections.Counter()
    data = []
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        src = r[1].strip()
        op = src.split()[0] if src else '?'
        if op.startswith('@'):
            op = src.split()[1]
        op = op.split('.')[0]
        cnt[op] += int(r[ie] or 0)
        for h in reasons:
            agg[op][h] += int(r[hdr.index(h)] or 0)
        data.append((int(r[si] or 0), src))
    tot = sum(sum(c.values()) for c in agg.values())
    print('samples', tot)
    for op, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:12]:
        print(f"{op:10s} {100 * sum(c.values()) / tot:5.1f}%  exec={cnt[op]:>12d}  ", dict(c.most_common(4)))
    print()
    for s, src in sorted(data, key=lambda x: -x[0])[:top]:
        print(s, src[:90])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
