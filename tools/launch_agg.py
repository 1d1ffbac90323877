"""Aggregate an ncu launch list by kernel name."""
import collections
import sys

sys.path.insert(0, __file__.rsplit('/', 1)[0])
from launches import rows  # noqa: E402

for path in sys.argv[1:]:
    r = rows(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for i, name, us in r:
        k = name.split('(')[0].replace('void ', '')[:80]
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(v[1] for v in agg.values())
    print(path, f"total {tot/1000:.2f} ms")
    for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{us/1000:9.2f} ms {100*us/tot:5.1f}%  n={c:4d}  avg={us/c:9.1f} us  {k}")
