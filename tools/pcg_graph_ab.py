"""A/B of the graph-resident PCG loop (LS_TUNE_PCG_GRAPH) on BASELINE configs 2 and 5 (p=2).

    python tools/pcg_graph_ab.py
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_10026_b200 as ls  # noqa: E402

for d, p, ne, kind in ((2, 3, 64, 0), (3, 3, 16, 1), (3, 2, 96, 1)):
    c = ls.Context(d, p, [ne] * (d + 1))
    s = torch.cuda.Stream()
    c.set_stream(s)
    b = c.rhs(kind)
    torch.cuda.synchronize()
    out = {"d": d, "p": p, "n_el": ne, "N": c.N}
    for g in (0, 1):
        c.tune(5, g)
        c.pcg(b, tol=1e-8)
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, st = c.pcg(b, tol=1e-8)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        out[f"graph{g}_ms"] = sorted(ts)[2]
        out["iters"] = st["iters"]
    print(json.dumps(out), flush=True)
    c.close()
